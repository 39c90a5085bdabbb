"""CPU oracle for the HODLR hot path of arXiv:1403.6015 -- TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference``) may import this package.  The
product package ``paper_1403_6015_b200`` never imports it and shares no code
with it.  See ``hodlr_oracle.h`` for the step -> paper map.
"""
from .oracle import (OracleHODLR, OracleError, build_oracle, dense_check, kernel_value,
                     aca_dense, SE, MATERN32, MATERN52, EXP, IMQ, RQ, MQ, BIHARM, KERNELS)

__all__ = ["OracleHODLR", "OracleError", "build_oracle", "dense_check", "kernel_value",
           "aca_dense", "SE", "MATERN32", "MATERN52", "EXP", "IMQ", "RQ", "MQ", "BIHARM", "KERNELS"]
