"""ctypes loader for liboracle.so and its Q15 twin liboracle_twin.so (TEST INFRASTRUCTURE; see oracle/__init__.py).

Argument marshalling only: every step of the HODLR method (build, factor, log det, solve, log-likelihood, apply)
runs in hodlr_oracle.c.  The one composite helper here is OracleHODLR.predict (eq_reg1 / eq_reg2), which combines
the C solve with C kernel values and forms the final dot products with numpy; it is pinned against the dense GP
posterior in tests/test_oracle_pins.py.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "hodlr_oracle.c")
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_TWIN_PATH = os.path.join(_HERE, "liboracle_twin.so")
_lock = threading.Lock()
_libs = {}

SE, MATERN32, MATERN52, EXP, IMQ, RQ, MQ, BIHARM = 0, 1, 2, 3, 4, 5, 6, 7
KERNELS = {"se": SE, "matern32": MATERN32, "matern52": MATERN52, "exp": EXP, "imq": IMQ, "rq": RQ, "mq": MQ,
           "biharm": BIHARM}
STATUS = {0: "OK", 1: "EINVAL", 2: "ENOTPD", 3: "ERANKCAP", 4: "ESTATE", 5: "ENOMEM"}


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"oracle {STATUS.get(code, code)}: {msg}")
        self.code = code
        self.status = STATUS.get(code, str(code))


def build_oracle(force: bool = False, twin: bool = False) -> str:
    """Compile hodlr_oracle.c with gcc -O2 -ffp-contract=off (no BLAS/OpenMP); twin=True adds -DORACLE_TWIN
    (leaf LU + coupling-system Householder QR)."""
    path = _TWIN_PATH if twin else _LIB_PATH
    if force or not os.path.exists(path) or os.path.getmtime(path) < os.path.getmtime(_SRC) \
            or os.path.getmtime(path) < os.path.getmtime(os.path.join(_HERE, "hodlr_oracle.h")):
        tmp = path + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fPIC", "-shared", "-Wall",
                               *(["-DORACLE_TWIN"] if twin else []), "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, path)
    return path


def _load(twin: bool = False):
    with _lock:
        if twin in _libs:
            return _libs[twin]
        lib = C.CDLL(build_oracle(twin=twin))
        P, I64, I32, D = C.c_void_p, C.c_int64, C.c_int, C.c_double
        lib.oracle_kernel.argtypes = [I32, P, D]; lib.oracle_kernel.restype = D
        lib.oracle_kernel_r2.argtypes = [I32, P, D]; lib.oracle_kernel_r2.restype = D
        lib.oracle_build_nd.argtypes = [P, I64, I32, I32, P, D, P, I32, D, I32, P]; lib.oracle_build_nd.restype = I32
        lib.oracle_dense_nd.argtypes = [P, I64, I32, I32, P, D, P, P, P, P]; lib.oracle_dense_nd.restype = I32
        lib.oracle_dim.argtypes = [P]; lib.oracle_dim.restype = I32
        lib.oracle_aca_dense.argtypes = [P, I64, I64, I64, D, I32, P, P, P]; lib.oracle_aca_dense.restype = I32
        lib.oracle_build.argtypes = [P, I64, I32, P, D, I32, D, I32, P]; lib.oracle_build.restype = I32
        lib.oracle_build_noise.argtypes = [P, I64, I32, P, D, P, I32, D, I32, P]; lib.oracle_build_noise.restype = I32
        lib.oracle_dense_noise.argtypes = [P, I64, I32, P, D, P, P, P, P]; lib.oracle_dense_noise.restype = I32
        for f in ("oracle_factor",):
            getattr(lib, f).argtypes = [P]; getattr(lib, f).restype = I32
        lib.oracle_logdet.argtypes = [P, P]; lib.oracle_logdet.restype = I32
        lib.oracle_logdet_sign.argtypes = [P, P, P]; lib.oracle_logdet_sign.restype = I32
        lib.oracle_solve.argtypes = [P, P, P, I64, I64]; lib.oracle_solve.restype = I32
        lib.oracle_gp_loglik.argtypes = [P, P, P]; lib.oracle_gp_loglik.restype = I32
        lib.oracle_apply.argtypes = [P, P, P]; lib.oracle_apply.restype = I32
        lib.oracle_kappa.argtypes = [P]; lib.oracle_kappa.restype = I32
        lib.oracle_num_nodes.argtypes = [P]; lib.oracle_num_nodes.restype = I64
        for f in ("oracle_get_perm", "oracle_get_sorted", "oracle_get_ranks"):
            getattr(lib, f).argtypes = [P, P]; getattr(lib, f).restype = I32
        lib.oracle_get_tree.argtypes = [P, P, P]; lib.oracle_get_tree.restype = I32
        lib.oracle_get_factors.argtypes = [P, I64, P, P]; lib.oracle_get_factors.restype = I32
        lib.oracle_get_logdet_parts.argtypes = [P, P, P]; lib.oracle_get_logdet_parts.restype = I32
        lib.oracle_free.argtypes = [P]; lib.oracle_free.restype = None
        lib.oracle_last_error.argtypes = []; lib.oracle_last_error.restype = C.c_char_p
        lib.oracle_dense.argtypes = [P, I64, I32, P, D, P, P, P]; lib.oracle_dense.restype = I32
        lib.oracle_residual_rows.argtypes = [P, P, P, P, I64, P]; lib.oracle_residual_rows.restype = I32
        _libs[twin] = lib
        return lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def _check(lib, code):
    if code != 0:
        raise OracleError(code, lib.oracle_last_error().decode())


def kernel_value(kernel: int, theta, d: float) -> float:
    lib = _load()
    th = np.ascontiguousarray(theta, dtype=np.float64)
    return lib.oracle_kernel(int(kernel), _ptr(th), float(d))


def aca_dense(A: np.ndarray, eps: float, cap: int | None = None):
    """O4 on an explicit dense block; returns (U, V, rank)."""
    lib = _load()
    A = np.asfortranarray(A, dtype=np.float64)
    m1, m2 = A.shape
    cap = min(m1, m2) if cap is None else cap
    U = np.zeros((cap, m1)); V = np.zeros((cap, m2)); r = C.c_int(0)
    _check(lib, lib.oracle_aca_dense(_ptr(A), m1, m2, m1, float(eps), int(cap), _ptr(U), _ptr(V), C.byref(r)))
    k = r.value
    return U[:k].T.copy(), V[:k].T.copy(), k


def kernel_value_r2(kernel: int, theta, r2: float) -> float:
    """O3 for d-dimensional points: k as a function of the squared distance r2 (NEXT-3)."""
    lib = _load()
    th = np.ascontiguousarray(theta, dtype=np.float64)
    return lib.oracle_kernel_r2(int(kernel), _ptr(th), float(r2))


def _points(x):
    """(n,) or (n, d) -> contiguous float64 (n, d) array and d."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    if x.ndim == 1:
        return x, 1
    return x, int(x.shape[1])


def dense_check(x, kernel: int, theta, sigma2: float, y=None, noise=None):
    """O11: dense Cholesky log det (+ solve).  Returns (logdet, x or None).  noise: heteroscedastic sigma_i^2 - sigma2.
    x: (n,) or (n, d) points."""
    lib = _load()
    x, dim = _points(x)
    nz = None if noise is None else np.ascontiguousarray(noise, dtype=np.float64)
    th = np.ascontiguousarray(theta, dtype=np.float64)
    ld = C.c_double(0.0)
    out = None
    if y is not None:
        y = np.ascontiguousarray(y, dtype=np.float64)
        out = np.zeros_like(y)
    _check(lib, lib.oracle_dense_nd(_ptr(x), x.shape[0], dim, int(kernel), _ptr(th), float(sigma2),
                                    _ptr(nz) if nz is not None else None, _ptr(y) if y is not None else None,
                                    C.byref(ld), _ptr(out) if out is not None else None))
    return ld.value, out


class OracleHODLR:
    """build -> factor -> {logdet, solve, gp_loglik}*, host memory, original point order."""

    def __init__(self, x, kernel: int, theta, sigma2: float, leaf: int, eps: float, rank_cap: int = 0,
                 twin: bool = False, noise=None):
        """x: (n,) points, or (n, d) for d-dimensional inputs (kd ordering, NEXT-3).  noise: optional heteroscedastic
        part, C_ii = sigma2 + noise_i."""
        self._lib = _load(twin)
        self.twin = twin
        self.x, self.dim = _points(x)
        self.n = self.x.shape[0]
        self.kernel, self.theta = int(kernel), tuple(float(v) for v in theta)
        th = np.ascontiguousarray(theta, dtype=np.float64)
        h = C.c_void_p(0)
        self._noise = None if noise is None else np.ascontiguousarray(noise, dtype=np.float64)
        _check(self._lib, self._lib.oracle_build_nd(_ptr(self.x), self.n, self.dim, int(kernel), _ptr(th),
                                                    float(sigma2), _ptr(self._noise) if self._noise is not None else None,
                                                    int(leaf), float(eps), int(rank_cap), C.byref(h)))
        self._h = h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            self._lib.oracle_free(h)
            self._h = None

    def factor(self):
        _check(self._lib, self._lib.oracle_factor(self._h))
        return self

    def logdet(self) -> float:
        v = C.c_double(0.0)
        _check(self._lib, self._lib.oracle_logdet(self._h, C.byref(v)))
        return v.value

    def logdet_sign(self):
        """(log |det C|, sign of det C) -- the kernels that are not SPD (MQ, BIHARM) may have det C < 0."""
        v = C.c_double(0.0); sg = C.c_int(0)
        _check(self._lib, self._lib.oracle_logdet_sign(self._h, C.byref(v), C.byref(sg)))
        return v.value, sg.value

    def solve(self, y):
        y = np.asarray(y, dtype=np.float64)
        one = y.ndim == 1
        Y = np.asfortranarray(y.reshape(self.n, -1))
        X = np.zeros_like(Y, order="F")
        _check(self._lib, self._lib.oracle_solve(self._h, _ptr(Y), _ptr(X), Y.shape[1], self.n))
        return X[:, 0].copy() if one else X

    def gp_loglik(self, y) -> float:
        y = np.ascontiguousarray(y, dtype=np.float64)
        v = C.c_double(0.0)
        _check(self._lib, self._lib.oracle_gp_loglik(self._h, _ptr(y), C.byref(v)))
        return v.value

    def apply(self, v):
        v = np.ascontiguousarray(v, dtype=np.float64)
        out = np.zeros_like(v)
        _check(self._lib, self._lib.oracle_apply(self._h, _ptr(v), _ptr(out)))
        return out

    def predict(self, y, xt, variance: bool = True):
        """GP prediction at test points xt (eq_reg1 / eq_reg2) with this oracle's HODLR solve:
        mean_j = k(xt_j, x) C^{-1} y; var_j = k(xt_j, xt_j) - k(xt_j, x) C^{-1} k(x, xt_j) (latent f, sigma^2 not
        added).  Cross-covariances entry by entry from oracle_kernel (Table I); plain loops,
        small cases only.  Requires factor()."""
        xt = np.asarray(xt, dtype=np.float64)
        alpha = self.solve(y)
        if self.dim == 1:
            Ks = np.array([[kernel_value(self.kernel, self.theta, float(t - xi)) for xi in self.x] for t in xt])
        else:
            xt = xt.reshape(-1, self.dim)
            Ks = np.array([[kernel_value_r2(self.kernel, self.theta, float(sum((t[k] - xi[k]) * (t[k] - xi[k])
                                                                                for k in range(self.dim))))
                            for xi in self.x] for t in xt])
        mean = Ks @ alpha
        if not variance:
            return mean, None
        var = np.array([kernel_value(self.kernel, self.theta, 0.0) - Ks[j] @ self.solve(Ks[j])
                        for j in range(Ks.shape[0])])
        return mean, var

    def residual_rows(self, xsol, y, rows):
        """(C x - y)[rows] with C assembled entry by entry in C (original order)."""
        xsol = np.ascontiguousarray(xsol, dtype=np.float64); y = np.ascontiguousarray(y, dtype=np.float64)
        rows = np.ascontiguousarray(rows, dtype=np.int64)
        out = np.zeros(rows.size)
        _check(self._lib, self._lib.oracle_residual_rows(self._h, _ptr(xsol), _ptr(y), _ptr(rows), rows.size, _ptr(out)))
        return out

    @property
    def kappa(self) -> int:
        return self._lib.oracle_kappa(self._h)

    def perm(self):
        p = np.zeros(self.n, dtype=np.int64)
        self._lib.oracle_get_perm(self._h, _ptr(p))
        return p

    def sorted_x(self):
        p = np.zeros(self.n * self.dim)
        self._lib.oracle_get_sorted(self._h, _ptr(p))
        return p if self.dim == 1 else p.reshape(self.n, self.dim)

    def tree(self):
        nn = self._lib.oracle_num_nodes(self._h)
        lo = np.zeros(nn, dtype=np.int64); hi = np.zeros(nn, dtype=np.int64)
        self._lib.oracle_get_tree(self._h, _ptr(lo), _ptr(hi))
        return lo, hi

    def ranks(self):
        ni = (1 << self.kappa) - 1
        r = np.zeros(max(ni, 1), dtype=np.int32)
        self._lib.oracle_get_ranks(self._h, _ptr(r))
        return r[:ni]

    def factors(self, node: int):
        lo, hi = self.tree()
        m1 = hi[2 * node + 1] - lo[2 * node + 1]; m2 = hi[2 * node + 2] - lo[2 * node + 2]
        r = int(self.ranks()[node])
        U = np.zeros((max(r, 1), m1)); V = np.zeros((max(r, 1), m2))
        _check(self._lib, self._lib.oracle_get_factors(self._h, node, _ptr(U), _ptr(V)))
        return U[:r].T.copy(), V[:r].T.copy()

    def logdet_parts(self):
        nl = 1 << self.kappa; ni = nl - 1
        a = np.zeros(nl); b = np.zeros(max(ni, 1))
        _check(self._lib, self._lib.oracle_get_logdet_parts(self._h, _ptr(a), _ptr(b)))
        return a, b[:ni]
