"""Parity at the hardest full-size cases (test tooling): cfg3 n = 2^20 at eps = 1e-12 and the 8 extreme config-4
settings at n = 131072, GPU vs oracle (log det, solve) with the Q15 twin floor of each config-4 setting.
python tools/parity_hard.py [out.json]"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1403_6015_b200 import inputs
import paper_1403_6015_b200.hodlr as hb
from oracle import OracleHODLR

cases = []
cfg = inputs.CONFIGS["cfg3"]
cases.append(("cfg3-full", inputs.points(cfg), inputs.rhs(cfg), cfg.kernel, cfg.theta, cfg.sigma2, cfg.leaf))
c4 = inputs.CONFIGS["cfg4"]
ell, s2 = inputs.sweep_settings(c4)
x4, y4 = inputs.points(c4), inputs.rhs(c4)
for k in [12, 17, 45, 36, 40, 43, 10, 15]:
    cases.append((f"cfg4-{k}", x4, y4, c4.kernel, (1.0, ell[k]), s2[k], c4.leaf))
out = []
for name, x, y, kern, th, sg, leaf in cases:
    o = OracleHODLR(x, kern, th, sg, leaf, 1e-12).factor()
    ld_o, x_o = o.logdet(), o.solve(y)
    floor = None
    if name.startswith("cfg4"):
        t = OracleHODLR(x, kern, th, sg, leaf, 1e-12, twin=True).factor()
        floor = float(np.linalg.norm(t.solve(y) - x_o) / np.linalg.norm(x_o))
    xd, yd = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
    g = hb.HODLR(xd, kern, th, sg, leaf, 1e-12).factor()
    ld_g, x_g = g.logdet(), g.solve(yd).cpu().numpy()
    g.close()
    r = {"case": name, "logdet_rel": abs(ld_g - ld_o) / abs(ld_o),
         "solve_rel": float(np.linalg.norm(x_g - x_o) / np.linalg.norm(x_o)), "twin_floor": floor}
    out.append(r)
    print(json.dumps(r), flush=True)
if len(sys.argv) > 1:
    json.dump(out, open(sys.argv[1], "w"), indent=1)
