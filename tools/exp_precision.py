"""Experiment: GPU-vs-oracle parity as a function of HODLR_TREE_PLAIN_FROM (depths >= that value run
the coupling-tree Schur updates in plain double).  Test tooling: prints one line per case.
HODLR_TREE_PLAIN_FROM=<d> python tools/exp_precision.py [full]   (the env var is read once per process)"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1403_6015_b200 import inputs
import paper_1403_6015_b200.hodlr as hb
from oracle import OracleHODLR

CASES = [("cfg3", 1 << 16, None), ("cfg1", 2048, None), ("cfg2", 65536, None), ("cfg4", 1 << 14, (2.0, 1e-4)),
         ("cfg4", 1 << 14, (0.05, 1e-4))]
if len(sys.argv) > 1 and sys.argv[1] == "full":
    CASES = [("cfg3", 1 << 20, None), ("cfg4", 1 << 17, (2.0, 1e-4))]
cache = "/tmp/exp_oracle"
os.makedirs(cache, exist_ok=True)
for name, n, over in CASES:
    cfg = inputs.scaled(inputs.CONFIGS[name], n)
    if name == "cfg4":
        ell, s2 = over
        theta, sigma2 = (cfg.a, ell), s2
    else:
        theta, sigma2 = cfg.theta, cfg.sigma2
    x = inputs.points(cfg); y = inputs.rhs(cfg)
    key = f"{cache}/{name}_{n}_{over}.npz"
    if os.path.exists(key):
        z = np.load(key); ld_o = float(z["ld"]); x_o = z["x"]
    else:
        o = OracleHODLR(x, cfg.kernel, theta, sigma2, cfg.leaf, 1e-12).factor()
        ld_o = o.logdet(); x_o = o.solve(y); np.savez(key, ld=ld_o, x=x_o)
    g = hb.HODLR(torch.from_numpy(x).cuda(), cfg.kernel, theta, sigma2, cfg.leaf, 1e-12).factor()
    ld_g = g.logdet(); x_g = g.solve(torch.from_numpy(y).cuda()).cpu().numpy()
    print(f"plain_from={os.environ.get('HODLR_TREE_PLAIN_FROM','-')} {name} n={n} {over}: logdet rel "
          f"{abs(ld_g-ld_o)/abs(ld_o):.2e} solve rel {np.linalg.norm(x_g-x_o)/np.linalg.norm(x_o):.2e}", flush=True)
