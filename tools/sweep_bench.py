"""Config 4 (BASELINE.json): 64 (ell, sigma2) settings, n = 131072, Matern-5/2, leaf 64, eps = 1e-10 through
gp_loglik_sweep on one GPU (batched handles); wall time per sweep and the per-family device times of one batched
factorization.  python tools/sweep_bench.py [reps]"""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1403_6015_b200 import inputs
import paper_1403_6015_b200.hodlr as hb
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
cfg = inputs.CONFIGS["cfg4"]
ell, s2 = inputs.sweep_settings(cfg)
x = torch.from_numpy(inputs.points(cfg)).cuda(); y = torch.from_numpy(inputs.rhs(cfg)).cuda()
th = np.stack([np.full(cfg.sweep, cfg.a), ell], 1)
for _ in range(2):
    hb.gp_loglik_sweep(x, y, cfg.kernel, th, s2, cfg.leaf, cfg.eps)     # warm-up (allocations, plans)
ts = []
for _ in range(reps):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    v = hb.gp_loglik_sweep(x, y, cfg.kernel, th, s2, cfg.leaf, cfg.eps)
    torch.cuda.synchronize(); ts.append(time.perf_counter() - t0)
t = float(np.median(ts))
print(f"batched sweep: {1e3 * t:.2f} ms per 64-setting sweep (median of {reps}: {[round(1e3 * a, 2) for a in ts]}), "
      f"{cfg.sweep * cfg.n / t:.3e} points/s; loglik range [{v.min():.6e}, {v.max():.6e}]", flush=True)
g = hb.HODLRBatch(x, cfg.kernel, th, s2, cfg.leaf, cfg.eps)
g.factor_solve(y.repeat(cfg.sweep), solve=False)
info = g.info(); g.close()
print("one batched factorization, kernel ms:", {k: round(v, 3) for k, v in info["kernel_ms"].items()},
      "kappa", info["kappa"], "max ranks", info["max_rank_by_depth"])
print(json.dumps({"config": "cfg4 sweep (batched)", "n": cfg.n, "settings": cfg.sweep, "ms_per_sweep": 1e3 * t,
                  "ms_samples": [1e3 * a for a in ts], "kernel_ms": info["kernel_ms"]}))
