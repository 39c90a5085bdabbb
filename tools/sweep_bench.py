"""Config 4 (BASELINE.json): 64 (ell, sigma2) settings, n = 131072, Matern-5/2, leaf 64, eps = 1e-10 through
gp_loglik_sweep on one GPU; wall time per sweep for several worker counts.  python tools/sweep_bench.py"""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1403_6015_b200 import inputs
import paper_1403_6015_b200.hodlr as hb
cfg = inputs.CONFIGS["cfg4"]
ell, s2 = inputs.sweep_settings(cfg)
x = torch.from_numpy(inputs.points(cfg)).cuda(); y = torch.from_numpy(inputs.rhs(cfg)).cuda()
th = np.stack([np.full(cfg.sweep, cfg.a), ell], 1)
out = {}
for w in [1, 2, 4, 8]:
    hb.gp_loglik_sweep(x, y, cfg.kernel, th, s2, cfg.leaf, cfg.eps, workers=w)     # warm-up
    torch.cuda.synchronize(); t0 = time.perf_counter()
    reps = 3
    for _ in range(reps):
        v = hb.gp_loglik_sweep(x, y, cfg.kernel, th, s2, cfg.leaf, cfg.eps, workers=w)
    torch.cuda.synchronize(); t = (time.perf_counter() - t0) / reps
    out[w] = t
    print(f"workers={w}: {1e3 * t:.1f} ms per 64-setting sweep, {cfg.sweep / t:.0f} settings/s, "
          f"{cfg.sweep * cfg.n / t:.3e} points/s; loglik range [{v.min():.6e}, {v.max():.6e}]", flush=True)
print(json.dumps({"config": "cfg4 sweep", "n": cfg.n, "settings": cfg.sweep, "ms_per_sweep": {k: 1e3 * v for k, v in out.items()}}))
