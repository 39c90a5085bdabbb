"""B200-native HODLR factorization / log det / solve / GP log-likelihood (arXiv:1403.6015).

The hot path lives in libhodlr_b200.so (hand-written CUDA for sm_100a behind the
C-ABI of include/hodlr.h).  ``paper_1403_6015_b200.hodlr`` is the thin ctypes
binding; ``inputs`` holds the seeded synthetic workloads.  Submodules are loaded
lazily so that importing ``inputs`` does not need torch or a GPU.
"""
import importlib

__all__ = ["hodlr", "inputs", "build"]


def __getattr__(name):
    if name in __all__:
        return importlib.import_module(f".{name}", __name__)
    raise AttributeError(name)
