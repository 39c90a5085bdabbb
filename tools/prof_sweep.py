"""One batched config-4 factorization (64 settings, hodlr_build_batch + hodlr_factor_solve + results), for ncu runs
and per-family timing.  python tools/prof_sweep.py [reps]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1403_6015_b200 import inputs
import paper_1403_6015_b200.hodlr as hb
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 1
cfg = inputs.CONFIGS["cfg4"]
ell, s2 = inputs.sweep_settings(cfg)
x = torch.from_numpy(inputs.points(cfg)).cuda(); y = torch.from_numpy(inputs.rhs(cfg)).cuda().repeat(cfg.sweep)
th = np.stack([np.full(cfg.sweep, cfg.a), ell], 1)
for _ in range(reps):
    g = hb.HODLRBatch(x, cfg.kernel, th, s2, cfg.leaf, cfg.eps)
    g.factor_solve(y, solve=False)
    ld, q = g.results()
    info = g.info(); g.close()
torch.cuda.synchronize()
print("kernel_ms", {k: round(v, 3) for k, v in info["kernel_ms"].items() if v})
