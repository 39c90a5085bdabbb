"""Timing of one build+factor+logdet+solve at a given config/eps (e.g. the parity epsilon 1e-12).
python tools/eps_timing.py cfg3 1e-12"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1403_6015_b200 import inputs
import paper_1403_6015_b200.hodlr as hb
cfg = inputs.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg3"]
eps = float(sys.argv[2]) if len(sys.argv) > 2 else cfg.eps
n = int(sys.argv[3]) if len(sys.argv) > 3 else cfg.n
cfg = inputs.scaled(cfg, n)
x = torch.from_numpy(inputs.points(cfg)).cuda(); y = torch.from_numpy(inputs.rhs(cfg)).cuda()
for rep in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    h = hb.HODLR(x, cfg.kernel, cfg.theta, cfg.sigma2, cfg.leaf, eps).factor()
    ld = h.logdet(); s = h.solve(y); torch.cuda.synchronize(); t = time.perf_counter() - t0
    inf = h.info(); h.close()
print(f"{cfg.name} n={n} eps={eps}: K={inf['K']} {1e3 * t:.2f} ms wall, families "
      f"{ {k: round(v / 3, 2) for k, v in inf['kernel_ms'].items() if v > 0} }")
