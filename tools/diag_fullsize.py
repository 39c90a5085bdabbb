"""Diagnostic (test tooling): full-size cfg3 at eps = 1e-12 -- GPU vs oracle solve difference, ACA rank
mismatches, and the exact relative residuals ||C x - y|| / ||y|| of both solutions from a dense
chunked matvec on the GPU (plain torch, fp64).  python tools/diag_fullsize.py [cfg] [n] [eps]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1403_6015_b200 import inputs
import paper_1403_6015_b200.hodlr as hb
from oracle import OracleHODLR

name = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 1 << 20
eps = float(sys.argv[3]) if len(sys.argv) > 3 else 1e-12
cfg = inputs.scaled(inputs.CONFIGS[name], n)
x = inputs.points(cfg); y = inputs.rhs(cfg)


def dense_residual(xv, sol):
    xs = torch.from_numpy(xv).cuda(); s = torch.from_numpy(sol).cuda(); yy = torch.from_numpy(y).cuda()
    r = torch.empty_like(s)
    c = 1.0 / (2 * cfg.ell ** 2)
    for i0 in range(0, n, 256):
        d = xs[i0:i0 + 256, None] - xs[None, :]
        if cfg.kernel == 0:
            blk = torch.exp(-(d * d) * c) * cfg.a ** 2
        else:
            sc = (3.0 if cfg.kernel == 1 else 5.0) ** 0.5 / cfg.ell
            t = d.abs() * sc
            blk = (1 + t) * torch.exp(-t) if cfg.kernel == 1 else (1 + t + t * t / 3) * torch.exp(-t)
            blk = blk * cfg.a ** 2
        r[i0:i0 + 256] = blk @ s
    r += cfg.sigma2 * s
    return float(torch.linalg.norm(r - yy) / torch.linalg.norm(yy))


t0 = time.time()
o = OracleHODLR(x, cfg.kernel, cfg.theta, cfg.sigma2, cfg.leaf, eps).factor()
ld_o = o.logdet(); x_o = o.solve(y); r_o = o.ranks()
t1 = time.time()
g = hb.HODLR(torch.from_numpy(x).cuda(), cfg.kernel, cfg.theta, cfg.sigma2, cfg.leaf, eps).factor()
ld_g = g.logdet(); x_g = g.solve(torch.from_numpy(y).cuda()).cpu().numpy()
_, _, r_g = g.tree()
mism = np.nonzero(r_g != r_o)[0]
print(f"{name} n={n} eps={eps}: oracle {t1 - t0:.1f}s; logdet rel {abs(ld_g - ld_o) / abs(ld_o):.2e}; "
      f"solve rel {np.linalg.norm(x_g - x_o) / np.linalg.norm(x_o):.2e}; rank mismatches {len(mism)} of {len(r_o)}"
      f" (depths {sorted(set(int(np.log2(b + 1)) for b in mism))[:10]})", flush=True)
print(f"  residual ||Cx-y||/||y||: gpu {dense_residual(x, x_g):.2e} oracle {dense_residual(x, x_o):.2e}", flush=True)
for b in mism[:40]:
    print(f"    block {b} depth {int(np.log2(b + 1))}: oracle {r_o[b]} gpu {r_g[b]}")
g.close()
# the same GPU factorization with the oracle's per-block ranks (hodlr_opts.forced_ranks): arithmetic only
gf = hb.HODLR(torch.from_numpy(x).cuda(), cfg.kernel, cfg.theta, cfg.sigma2, cfg.leaf, eps, rank_cap=64,
              forced_ranks=r_o).factor()
ld_f = gf.logdet(); x_f = gf.solve(torch.from_numpy(y).cuda()).cpu().numpy()
_, _, r_f = gf.tree()
print(f"  forced ranks: equal {np.array_equal(r_f, r_o)}; logdet rel {abs(ld_f - ld_o) / abs(ld_o):.2e}; solve rel "
      f"{np.linalg.norm(x_f - x_o) / np.linalg.norm(x_o):.2e}; max elementwise {np.abs(x_f - x_o).max() / np.abs(x_o).max():.2e};"
      f" residual {dense_residual(x, x_f):.2e}", flush=True)
gf.close()
t2 = time.time()
tw = OracleHODLR(x, cfg.kernel, cfg.theta, cfg.sigma2, cfg.leaf, eps, twin=True).factor()
x_t = tw.solve(y)
print(f"  twin ({time.time() - t2:.1f}s): floor solve rel {np.linalg.norm(x_t - x_o) / np.linalg.norm(x_o):.2e}; logdet rel "
      f"{abs(tw.logdet() - ld_o) / abs(ld_o):.2e}", flush=True)
