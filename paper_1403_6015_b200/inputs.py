"""Seeded synthetic inputs for the five BASELINE.json configs.

This module holds NO arithmetic of the method: it only draws the points,
right-hand sides and hyper-parameters with numpy's PCG64, in the order
x, then y (then config-5 duplicates / config-4 settings), as DESIGN.md
section 4 states.  Both the CUDA path and the oracle receive the same arrays.

The paper's workloads are synthetic uniform points (PAPER.md:1303-1308,
1454-1455); no public dataset is involved.
"""
from __future__ import annotations

import dataclasses

import numpy as np

SE, MATERN32, MATERN52 = 0, 1, 2


@dataclasses.dataclass(frozen=True)
class Config:
    name: str
    n: int
    lo: float
    hi: float
    kernel: int
    a: float
    ell: float
    sigma2: float
    leaf: int
    eps: float
    seed: int
    dup_frac: float = 0.0        # config 5: fraction of clustered duplicates (R14)
    dup_jitter: float = 0.0
    sweep: int = 0               # config 4: number of (ell, sigma2) settings

    @property
    def theta(self):
        return (self.a, self.ell)


CONFIGS = {
    "cfg1": Config("cfg1", 2048, 0.0, 1.0, SE, 1.0, 0.1, 1e-2, 64, 1e-12, 1),
    "cfg2": Config("cfg2", 65536, 0.0, 10.0, MATERN32, 1.0, 0.5, 1e-3, 64, 1e-12, 2),
    "cfg3": Config("cfg3", 1 << 20, 0.0, 100.0, SE, 1.0, 1.0, 1e-2, 128, 1e-10, 3),
    "cfg4": Config("cfg4", 131072, 0.0, 10.0, MATERN52, 1.0, float("nan"), float("nan"), 64, 1e-10, 4,
                   sweep=64),
    "cfg5": Config("cfg5", 1 << 23, 0.0, 1000.0, SE, 1.0, 2.0, 1e-2, 128, 1e-10, 5,
                   dup_frac=0.05, dup_jitter=1e-6),
}


def points(cfg: Config, n: int | None = None, sort: bool = True) -> np.ndarray:
    """x ~ U[lo, hi] (seeded), optionally with config-5 duplicates; sorted as the configs state."""
    n = cfg.n if n is None else n
    rng = np.random.default_rng(cfg.seed)
    if cfg.dup_frac > 0.0:
        ndup = int(np.floor(cfg.dup_frac * n))
        base = rng.uniform(cfg.lo, cfg.hi, n - ndup)
        _ = rng.standard_normal(n)                     # y is drawn second (keeps the draw order)
        src = rng.integers(0, n - ndup, ndup)
        jit = rng.uniform(-cfg.dup_jitter, cfg.dup_jitter, ndup)
        x = np.concatenate([base, base[src] + jit])
    else:
        x = rng.uniform(cfg.lo, cfg.hi, n)
    return np.sort(x) if sort else x


def rhs(cfg: Config, n: int | None = None) -> np.ndarray:
    """y ~ N(0, 1), drawn after x from the same stream."""
    n = cfg.n if n is None else n
    rng = np.random.default_rng(cfg.seed)
    if cfg.dup_frac > 0.0:
        ndup = int(np.floor(cfg.dup_frac * n))
        rng.uniform(cfg.lo, cfg.hi, n - ndup)
    else:
        rng.uniform(cfg.lo, cfg.hi, n)
    return rng.standard_normal(n)


def sweep_settings(cfg: Config, count: int | None = None, seed: int = 44):
    """Config 4: (ell, sigma2) pairs, ell log-uniform [0.05, 2], sigma2 log-uniform [1e-4, 1e-1]."""
    count = cfg.sweep if count is None else count
    rng = np.random.default_rng(seed)
    ell = np.exp(rng.uniform(np.log(0.05), np.log(2.0), count))
    s2 = np.exp(rng.uniform(np.log(1e-4), np.log(1e-1), count))
    return ell, s2


def scaled(cfg: Config, n: int) -> Config:
    """Same point density and kernel on a smaller n (interval shrunk in proportion)."""
    width = (cfg.hi - cfg.lo) * n / cfg.n
    return dataclasses.replace(cfg, n=n, hi=cfg.lo + width)


def rmse_model(n: int = 1024, seed: int = 56):
    """The sec. 5.6 regression data: x_j uniform in (-3, 3), y = sin(2x) + e^x / 8 + N(0, 1)
    (sigma_eps = 1), seeded.  Returns (x, y) in generation order (unsorted)."""
    rng = np.random.default_rng(seed)
    x = rng.uniform(-3.0, 3.0, n)
    y = np.sin(2.0 * x) + np.exp(x) / 8.0 + rng.standard_normal(n)
    return x, y


# NEXT-3 workloads (DESIGN.md section 4 / 9f): the shape of Table II's multi-dimensional columns -- "random uniformly
# distributed points" in a cube -- with the cube and length scale chosen so that the ranks meet
# eps within this build's rank cap (the paper's [-3, 3]^d with exp(-r^2) has ranks in the hundreds).
ND_CONFIGS = {
    #        d, half-side, kernel, (a, ell), sigma2, leaf, eps
    "nd2": (2, 0.5, SE, (1.0, 1.0), 1e-2, 128, 1e-10),
    "nd3": (3, 0.5, SE, (1.0, 4.0), 1e-2, 128, 1e-10),
}


def points_nd(n: int, d: int, seed: int, half: float = 0.5, grid: int = 0):
    """(x, y): n points uniform in [-half, half]^d (row-major (n, d)), then y ~ N(0, 1).  grid > 0 rounds every
    coordinate to a multiple of 1/grid (exact coordinate ties and duplicate points: the kd sort's tie rule and the
    ACA's duplicate-row rule)."""
    rng = np.random.default_rng(seed)
    x = rng.uniform(-half, half, (n, d))
    if grid > 0:
        x = np.round(x * grid) / grid
    y = rng.standard_normal(n)
    return x, y
