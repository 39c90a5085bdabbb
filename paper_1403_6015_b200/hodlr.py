"""Thin ctypes binding of include/hodlr.h (argument marshalling only).

Every step of the hot path runs in libhodlr_b200.so's CUDA kernels.  There is
no CPU fallback: if the library or a CUDA device is missing, calls raise.
PyTorch supplies device memory (tensors) and the stream.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

import torch

from . import build as _build

HODLR_SE, HODLR_MATERN32, HODLR_MATERN52, HODLR_EXP, HODLR_IMQ, HODLR_RQ = 0, 1, 2, 3, 4, 5
HODLR_MQ, HODLR_BIHARM = 6, 7      # not positive definite (hodlr.h, R20)
KERNELS = {"se": HODLR_SE, "matern32": HODLR_MATERN32, "matern52": HODLR_MATERN52, "exp": HODLR_EXP,
           "imq": HODLR_IMQ, "rq": HODLR_RQ, "mq": HODLR_MQ, "biharm": HODLR_BIHARM}
STATUS = {0: "OK", 1: "EINVAL", 2: "ENOTPD", 3: "ERANKCAP", 4: "ESTATE", 5: "ENOMEM", 6: "ECUDA", 7: "ENCCL"}

EXPORTS = ("hodlr_build", "hodlr_factor", "hodlr_factor_solve", "hodlr_cache_trim", "hodlr_logdet",
           "hodlr_logdet_sign", "hodlr_solve", "hodlr_apply", "gp_predict", "gp_loglik",
           "hodlr_info",
           "hodlr_get_order", "hodlr_get_tree", "hodlr_get_logdet_parts", "hodlr_free", "hodlr_last_error",
           "hodlr_version", "hodlr_launch_count", "hodlr_nccl_unique_id", "hodlr_group_create",
           "hodlr_group_destroy", "hodlr_group_mode", "hodlr_dist_plan", "gp_loglik_sweep", "hodlr_build_batch",
           "hodlr_batch_results", "hodlr_build_nd")


class HodlrError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"hodlr {STATUS.get(code, code)}: {msg}")
        self.code = code
        self.status = STATUS.get(code, str(code))


class hodlr_dist(C.Structure):
    _fields_ = [("rank", C.c_int32), ("nranks", C.c_int32), ("nccl_unique_id", C.c_void_p), ("group", C.c_void_p)]


class hodlr_opts(C.Structure):
    _fields_ = [("rank_cap", C.c_int32), ("flags", C.c_int32), ("forced_ranks", C.c_void_p), ("noise", C.c_void_p),
                ("reserved", C.c_int64 * 5)]


class hodlr_info_t(C.Structure):
    _fields_ = [("kappa", C.c_int32), ("leaf_min", C.c_int32), ("leaf_max", C.c_int32), ("K", C.c_int32),
                ("max_rank_by_depth", C.c_int32 * 64), ("mean_rank_by_depth", C.c_double * 64),
                ("factor_bytes", C.c_int64), ("t_build", C.c_double), ("t_factor", C.c_double),
                ("t_logdet", C.c_double), ("t_solve", C.c_double), ("rank_cap_hits", C.c_int64),
                ("aca_steps", C.c_int32), ("gpu_launches_last", C.c_int32),
                ("kernel_ms", C.c_double * 16), ("kernel_calls", C.c_int64 * 16),
                ("rank", C.c_int32), ("nranks", C.c_int32), ("split_depth", C.c_int32), ("pad_", C.c_int32)]

KERNEL_FAMILIES = ("sort", "aca", "leaf_factor", "coupling_tree", "solve", "unused5", "unused6", "leaf_chol")


_lib = None
_lock = threading.Lock()


def library_path() -> str:
    return _build.LIB


def load(build_if_missing: bool = True):
    """Load libhodlr_b200.so (building it with nvcc if missing).  Raises if unavailable."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        path = os.environ.get("HODLR_LIB") or _build.LIB   # HODLR_LIB: an alternative build (experiments)
        if not os.path.exists(path):
            if not build_if_missing:
                raise RuntimeError(f"{path} missing; run python -m paper_1403_6015_b200.build")
            _build.build()
        lib = C.CDLL(path)
        P, I64, I32, D = C.c_void_p, C.c_int64, C.c_int32, C.c_double
        lib.hodlr_build.argtypes = [P, I64, I32, P, D, I32, D, P, P, P, P]
        lib.hodlr_factor.argtypes = [P]
        lib.hodlr_factor_solve.argtypes = [P, P, P, P]; lib.hodlr_factor_solve.restype = I32
        lib.hodlr_cache_trim.argtypes = []; lib.hodlr_cache_trim.restype = None
        lib.hodlr_logdet.argtypes = [P, P]
        lib.hodlr_logdet_sign.argtypes = [P, P, P]
        lib.hodlr_solve.argtypes = [P, P, P, I64, I64]
        lib.hodlr_apply.argtypes = [P, P, P, I64, I64]
        lib.gp_predict.argtypes = [P, P, P, I64, P, P]
        lib.gp_loglik.argtypes = [P, P, P]
        lib.hodlr_info.argtypes = [P, P]
        lib.hodlr_get_order.argtypes = [P, P, P]
        lib.hodlr_get_tree.argtypes = [P, P, P, P]
        lib.hodlr_get_logdet_parts.argtypes = [P, P, P]
        for f in ("hodlr_build", "hodlr_factor", "hodlr_logdet", "hodlr_logdet_sign", "hodlr_solve", "hodlr_apply", "gp_predict", "gp_loglik",
                  "hodlr_info", "hodlr_get_order", "hodlr_get_tree", "hodlr_get_logdet_parts"):
            getattr(lib, f).restype = I32
        lib.hodlr_free.argtypes = [P]; lib.hodlr_free.restype = None
        lib.hodlr_last_error.argtypes = []; lib.hodlr_last_error.restype = C.c_char_p
        lib.hodlr_version.argtypes = []; lib.hodlr_version.restype = C.c_char_p
        lib.hodlr_launch_count.argtypes = []; lib.hodlr_launch_count.restype = C.c_int64
        lib.hodlr_nccl_unique_id.argtypes = [P]; lib.hodlr_nccl_unique_id.restype = I32
        lib.hodlr_group_create.argtypes = [I32, P]; lib.hodlr_group_create.restype = I32
        lib.hodlr_group_destroy.argtypes = [P]; lib.hodlr_group_destroy.restype = None
        lib.hodlr_group_mode.argtypes = [P, I32]; lib.hodlr_group_mode.restype = I32
        lib.hodlr_dist_plan.argtypes = [I64, I32, I32, I32, P, P, P, P, P, P]; lib.hodlr_dist_plan.restype = I32
        lib.gp_loglik_sweep.argtypes = [P, P, I64, I32, P, P, I32, I32, D, P, P, I32, P]
        lib.hodlr_build_batch.argtypes = [P, I64, I32, P, P, I32, I32, D, P, P, P]
        lib.hodlr_batch_results.argtypes = [P, P, P]
        lib.hodlr_build_nd.argtypes = [P, I64, I32, I32, P, D, I32, D, P, P, P]; lib.hodlr_build_nd.restype = I32
        lib.gp_loglik_sweep.restype = I32
        _lib = lib
        return lib


def _check(code: int):
    if code != 0:
        raise HodlrError(code, load().hodlr_last_error().decode())


def _dev_f64(t: torch.Tensor, name: str) -> torch.Tensor:
    if not isinstance(t, torch.Tensor) or t.device.type != "cuda" or t.dtype != torch.float64:
        raise TypeError(f"{name} must be a CUDA float64 tensor")
    return t.contiguous()


def _stream_ptr(stream) -> int:
    s = torch.cuda.current_stream() if stream is None else stream
    return int(s.cuda_stream)


# ------------------------------------------------------------------ C-ABI mirrors
def hodlr_build(x: torch.Tensor, kernel: int, theta, sigma2: float, leaf: int, eps: float,
                rank_cap: int = 0, stream=None, dist: "hodlr_dist | None" = None, forced_ranks=None,
                noise: "torch.Tensor | None" = None) -> int:
    """forced_ranks: optional int32 array of the internal nodes' ACA ranks (heap order) -- the parity test hook of
    hodlr_opts.forced_ranks.  noise: optional CUDA float64 (n,) heteroscedastic part of the diagonal."""
    lib = load()
    x = _dev_f64(x, "x")
    th = (C.c_double * 3)(float(theta[0]), float(theta[1]), float(theta[2]) if len(theta) > 2 else 0.0)
    opts = hodlr_opts(int(rank_cap))
    if forced_ranks is not None:
        import numpy as np
        fr = np.ascontiguousarray(forced_ranks, dtype=np.int32)
        opts.forced_ranks = fr.ctypes.data
    if noise is not None:
        noise = _dev_f64(noise, "noise")
        opts.noise = noise.data_ptr()
    h = C.c_void_p(0)
    _check(lib.hodlr_build(x.data_ptr(), x.numel(), int(kernel), th, float(sigma2), int(leaf), float(eps),
                           C.byref(dist) if dist is not None else None, C.byref(opts), _stream_ptr(stream),
                           C.byref(h)))
    return h.value


def hodlr_build_nd(x: torch.Tensor, kernel: int, theta, sigma2: float, leaf: int, eps: float,
                   rank_cap: int = 0, stream=None, forced_ranks=None, noise: "torch.Tensor | None" = None) -> int:
    """NEXT-3: x is a CUDA float64 (n, d) tensor of d-dimensional points (row-major), kd ordering (hodlr.h)."""
    lib = load()
    x = _dev_f64(x, "x")
    if x.dim() != 2:
        raise ValueError("hodlr_build_nd: x must be (n, d)")
    th = (C.c_double * 3)(float(theta[0]), float(theta[1]), float(theta[2]) if len(theta) > 2 else 0.0)
    opts = hodlr_opts(int(rank_cap))
    if forced_ranks is not None:
        import numpy as np
        fr = np.ascontiguousarray(forced_ranks, dtype=np.int32)
        opts.forced_ranks = fr.ctypes.data
    if noise is not None:
        noise = _dev_f64(noise, "noise")
        opts.noise = noise.data_ptr()
    h = C.c_void_p(0)
    _check(lib.hodlr_build_nd(x.data_ptr(), x.shape[0], x.shape[1], int(kernel), th, float(sigma2), int(leaf),
                              float(eps), C.byref(opts), _stream_ptr(stream), C.byref(h)))
    return h.value


def hodlr_build_batch(x: torch.Tensor, kernel: int, thetas, sigma2s, leaf: int, eps: float, rank_cap: int = 0,
                      stream=None, forced_ranks=None) -> int:
    """B = 2^t problems on the same points (hodlr_build_batch): thetas (B, 2) {a, ell} ((B, 3) for RQ), sigma2s (B,)."""
    import numpy as np
    lib = load()
    x = _dev_f64(x, "x")
    s2 = np.ascontiguousarray(np.asarray(sigma2s, dtype=np.float64).reshape(-1))
    th = np.ascontiguousarray(np.asarray(thetas, dtype=np.float64).reshape(s2.size, -1))
    opts = hodlr_opts(int(rank_cap))
    if forced_ranks is not None:
        fr = np.ascontiguousarray(forced_ranks, dtype=np.int32)
        opts.forced_ranks = fr.ctypes.data
    h = C.c_void_p(0)
    _check(lib.hodlr_build_batch(x.data_ptr(), x.numel(), int(kernel), th.ctypes.data, s2.ctypes.data, s2.size,
                                 int(leaf), float(eps), C.byref(opts), _stream_ptr(stream), C.byref(h)))
    return h.value


def hodlr_batch_results(h: int, nbatch: int, quad: bool = True):
    """Per-problem log det (and y_s^T C_s^{-1} y_s of the fused right-hand side): numpy arrays."""
    import numpy as np
    ld = np.zeros(nbatch); q = np.zeros(nbatch)
    _check(load().hodlr_batch_results(h, ld.ctypes.data, q.ctypes.data if quad else None))
    return (ld, q) if quad else ld


def hodlr_factor(h: int):
    _check(load().hodlr_factor(h))


def hodlr_factor_solve(h: int, y: torch.Tensor, solve: bool = True, out: "torch.Tensor | None" = None):
    """Fused factor + solve of one right-hand side: returns (C^{-1} y or None, y^T C^{-1} y).  out: optional
    contiguous float64 tensor of n entries for C^{-1} y -- on the device or in pinned host memory (then the solve
    kernel writes it directly: the device-to-host transfer overlaps the solve)."""
    lib = load()
    y = _dev_f64(y, "y")
    if out is not None:
        if out.dtype != torch.float64 or not out.is_contiguous() or out.numel() != y.numel() or \
                (out.device.type != "cuda" and not out.is_pinned()):
            raise TypeError("out must be a contiguous float64 CUDA or pinned CPU tensor of n entries")
        x = out
    else:
        x = torch.empty_like(y) if solve else None
    q = C.c_double(0.0)
    _check(lib.hodlr_factor_solve(h, y.data_ptr(), x.data_ptr() if x is not None else None, C.byref(q)))
    return x, q.value


def hodlr_cache_trim():
    load().hodlr_cache_trim()


def hodlr_logdet(h: int) -> float:
    v = C.c_double(0.0)
    _check(load().hodlr_logdet(h, C.byref(v)))
    return v.value


def hodlr_logdet_sign(h: int):
    """(log |det C|, sign of det C) -- the sign is -1 only for a kernel that is not positive definite."""
    v = C.c_double(0.0); sg = C.c_int32(0)
    _check(load().hodlr_logdet_sign(h, C.byref(v), C.byref(sg)))
    return v.value, sg.value


def hodlr_solve(h: int, y: torch.Tensor, x: torch.Tensor | None = None) -> torch.Tensor:
    """y: (n,) or (n, nrhs) CUDA float64 (column-major storage is made internally)."""
    lib = load()
    y = _dev_f64(y, "y")
    one = y.dim() == 1
    Y = y.reshape(y.shape[0], -1).t().contiguous()          # nrhs x n rows = column-major n x nrhs
    X = torch.empty_like(Y)
    _check(lib.hodlr_solve(h, Y.data_ptr(), X.data_ptr(), Y.shape[0], Y.shape[1]))
    out = X[0] if one else X.t()
    if x is not None:
        x.copy_(out)
        return x
    return out


def hodlr_apply(h: int, x: torch.Tensor) -> torch.Tensor:
    """y = C~ x of the compressed operator; x: (n,) or (n, nrhs) CUDA float64."""
    lib = load()
    x = _dev_f64(x, "x")
    one = x.dim() == 1
    X = x.reshape(x.shape[0], -1).t().contiguous()          # nrhs x n rows = column-major n x nrhs
    Y = torch.empty_like(X)
    _check(lib.hodlr_apply(h, X.data_ptr(), Y.data_ptr(), X.shape[0], X.shape[1]))
    return Y[0] if one else Y.t()


def gp_predict(h: int, y: torch.Tensor, xt: torch.Tensor, variance: bool = True):
    """Predictive mean (and latent variance) at test points xt (CUDA float64); returns (mean, var or None)."""
    lib = load()
    y = _dev_f64(y, "y"); xt = _dev_f64(xt, "xt")
    m = xt.shape[0] if xt.dim() == 2 else xt.numel()      # (m, d) test points on a d-dimensional handle
    mean = torch.empty(m, dtype=torch.float64, device=xt.device)
    var = torch.empty(m, dtype=torch.float64, device=xt.device) if variance else None
    _check(lib.gp_predict(h, y.data_ptr(), xt.data_ptr(), m, mean.data_ptr(),
                          var.data_ptr() if var is not None else None))
    return mean, var


def gp_loglik(h: int, y: torch.Tensor) -> float:
    y = _dev_f64(y, "y")
    v = C.c_double(0.0)
    _check(load().gp_loglik(h, y.data_ptr(), C.byref(v)))
    return v.value


def gp_loglik_sweep(x: torch.Tensor, y: torch.Tensor, kernel: int, thetas, sigma2s, leaf: int, eps: float,
                    dist=None, workers: int = 0, stream=None):
    """Config 4: log-likelihoods of B settings; thetas (B, 2) {a, ell}, sigma2s (B,).  Returns a numpy array."""
    import numpy as np
    lib = load()
    x = _dev_f64(x, "x"); y = _dev_f64(y, "y")
    th = np.ascontiguousarray(np.asarray(thetas, dtype=np.float64).reshape(-1, 2))
    s2 = np.ascontiguousarray(np.asarray(sigma2s, dtype=np.float64).reshape(-1))
    out = np.zeros(s2.size)
    ds = dist.struct() if dist is not None else None
    code = lib.gp_loglik_sweep(x.data_ptr(), y.data_ptr(), x.numel(), int(kernel), th.ctypes.data, s2.ctypes.data,
                               s2.size, int(leaf), float(eps), C.byref(ds) if ds is not None else None,
                               _stream_ptr(stream), int(workers), out.ctypes.data)
    if code != 0 and not np.all(np.isneginf(out) | np.isfinite(out)):
        _check(code)
    if code != 0:
        err = HodlrError(code, load().hodlr_last_error().decode())
        err.values = out
        raise err
    return out


def hodlr_info(h: int) -> dict:
    info = hodlr_info_t()
    _check(load().hodlr_info(h, C.byref(info)))
    k = info.kappa
    return {"kappa": k, "leaf_min": info.leaf_min, "leaf_max": info.leaf_max, "K": info.K,
            "max_rank_by_depth": list(info.max_rank_by_depth[1:k + 1]),
            "mean_rank_by_depth": list(info.mean_rank_by_depth[1:k + 1]),
            "factor_bytes": info.factor_bytes, "t_build": info.t_build, "t_factor": info.t_factor,
            "t_logdet": info.t_logdet, "t_solve": info.t_solve, "rank_cap_hits": info.rank_cap_hits,
            "aca_steps": info.aca_steps, "gpu_launches_last": info.gpu_launches_last,
            "kernel_ms": {f: info.kernel_ms[i] for i, f in enumerate(KERNEL_FAMILIES)},
            "kernel_calls": {f: info.kernel_calls[i] for i, f in enumerate(KERNEL_FAMILIES)},
            "rank": info.rank, "nranks": info.nranks, "split_depth": info.split_depth}


def hodlr_launch_count() -> int:
    return int(load().hodlr_launch_count())


def hodlr_free(h: int):
    if h:
        load().hodlr_free(h)


def hodlr_dist_plan(n: int, leaf: int, rank: int, nranks: int) -> dict:
    """Host-side shard plan (no device work): kappa, split depth t, owned sorted rows and leaves."""
    lib = load()
    k, t = C.c_int32(0), C.c_int32(0)
    rl, rh, ll, lh = C.c_int64(0), C.c_int64(0), C.c_int64(0), C.c_int64(0)
    _check(lib.hodlr_dist_plan(int(n), int(leaf), int(rank), int(nranks), C.byref(k), C.byref(t), C.byref(rl),
                               C.byref(rh), C.byref(ll), C.byref(lh)))
    return {"kappa": k.value, "t": t.value, "row_lo": rl.value, "row_hi": rh.value,
            "leaf_lo": ll.value, "leaf_hi": lh.value}


class HODLR:
    """build -> factor -> {logdet, solve, gp_loglik}* on one GPU; inputs are CUDA float64 tensors."""

    def __init__(self, x: torch.Tensor, kernel, theta, sigma2: float, leaf: int, eps: float,
                 rank_cap: int = 0, stream=None, dist=None, forced_ranks=None, noise=None):
        """dist: None (one GPU) or a paper_1403_6015_b200.dist.Dist (subtree sharding).  forced_ranks: parity test
        hook (hodlr_opts.forced_ranks)."""
        if isinstance(kernel, str):
            kernel = KERNELS[kernel]
        self._dist = dist                       # keeps the NCCL id / group alive
        if x.dim() == 2:                        # (n, d) points: hodlr_build_nd (NEXT-3, one GPU)
            if dist is not None:
                raise ValueError("HODLR: d-dimensional points run on one GPU (no dist)")
            self.n, self.dim = x.shape[0], x.shape[1]
            self._h = hodlr_build_nd(x, kernel, theta, sigma2, leaf, eps, rank_cap, stream, forced_ranks, noise)
            return
        self.n, self.dim = x.numel(), 1
        self._h = hodlr_build(x, kernel, theta, sigma2, leaf, eps, rank_cap, stream,
                              dist.struct() if dist is not None else None, forced_ranks, noise)

    def __del__(self):
        h = getattr(self, "_h", 0)
        if h:
            try:
                hodlr_free(h)
            except TypeError:                   # interpreter shutdown: module globals already cleared
                pass
            self._h = 0

    def close(self):
        self.__del__()

    def factor(self):
        hodlr_factor(self._h)
        return self

    def factor_solve(self, y: torch.Tensor, solve: bool = True, out: "torch.Tensor | None" = None):
        """Factor with y fused in; returns (C^{-1} y or None, y^T C^{-1} y).  The handle is then factored.
        out: optional destination of C^{-1} y (CUDA or pinned CPU tensor)."""
        return hodlr_factor_solve(self._h, y, solve, out)

    def logdet(self) -> float:
        return hodlr_logdet(self._h)

    def logdet_sign(self):
        return hodlr_logdet_sign(self._h)

    def solve(self, y: torch.Tensor) -> torch.Tensor:
        return hodlr_solve(self._h, y)

    def gp_loglik(self, y: torch.Tensor) -> float:
        return gp_loglik(self._h, y)

    def apply(self, x: torch.Tensor) -> torch.Tensor:
        return hodlr_apply(self._h, x)

    def predict(self, y: torch.Tensor, xt: torch.Tensor, variance: bool = True):
        return gp_predict(self._h, y, xt, variance)

    def info(self) -> dict:
        return hodlr_info(self._h)

    def order(self):
        """(sorted points, perm): points (n,) for 1-D, (n, d) for a d-dimensional handle."""
        dim = getattr(self, "dim", 1)
        xs = torch.empty(self.n * dim, dtype=torch.float64, device="cuda")
        perm = torch.empty(self.n, dtype=torch.int64, device="cuda")
        _check(load().hodlr_get_order(self._h, xs.data_ptr(), perm.data_ptr()))
        if dim > 1:
            xs = xs.view(dim, self.n).t().contiguous()     # coordinate-major on the device -> (n, d)
        return xs, perm

    def tree(self):
        import numpy as np
        k = self.info()["kappa"]
        nn = (1 << (k + 1)) - 1; ni = (1 << k) - 1
        lo = np.zeros(nn, dtype=np.int64); hi = np.zeros(nn, dtype=np.int64); r = np.zeros(max(ni, 1), dtype=np.int32)
        _check(load().hodlr_get_tree(self._h, lo.ctypes.data, hi.ctypes.data, r.ctypes.data))
        return lo, hi, r[:ni]

    def logdet_parts(self):
        import numpy as np
        k = self.info()["kappa"]
        a = np.zeros(1 << k); b = np.zeros(max((1 << k) - 1, 1))
        _check(load().hodlr_get_logdet_parts(self._h, a.ctypes.data, b.ctypes.data))
        return a, b[:(1 << k) - 1]


class HODLRBatch(HODLR):
    """B = 2^t problems (thetas[s], sigma2s[s]) on the same points x, held as one block-diagonal handle of order
    B n (hodlr_build_batch); vectors are problem-major (B n,)."""

    def __init__(self, x: torch.Tensor, kernel, thetas, sigma2s, leaf: int, eps: float, rank_cap: int = 0,
                 stream=None, forced_ranks=None):
        if isinstance(kernel, str):
            kernel = KERNELS[kernel]
        import numpy as np
        self.nbatch = int(np.asarray(sigma2s).size)
        self.n = x.numel() * self.nbatch
        self._dist = None
        self._h = hodlr_build_batch(x, kernel, thetas, sigma2s, leaf, eps, rank_cap, stream, forced_ranks)

    def results(self, quad: bool = True):
        return hodlr_batch_results(self._h, self.nbatch, quad)
