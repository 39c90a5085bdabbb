"""Timing experiment: ACA phase time with only some depth loops enabled (HODLR_ACA_GROUP_MASK, results invalid
for the disabled depths).  Each mask runs in its own process.  python tools/aca_groups.py <mask>"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1403_6015_b200 import inputs
import paper_1403_6015_b200.hodlr as hb
cfg = inputs.CONFIGS["cfg3"]
x = torch.from_numpy(inputs.points(cfg)).cuda()
ts = []
for rep in range(4):
    h = hb.HODLR(x, cfg.kernel, cfg.theta, cfg.sigma2, cfg.leaf, cfg.eps)
    inf = h.info(); h.close()
    ts.append(inf["kernel_ms"]["aca"])
print(f"mask={os.environ.get('HODLR_ACA_GROUP_MASK')}: aca phase ms {[round(t, 3) for t in ts[1:]]}", flush=True)
