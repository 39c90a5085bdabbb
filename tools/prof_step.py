"""One full hot-path step (build, factor_solve, logdet) on a BASELINE config, for ncu runs.
python tools/prof_step.py [cfg3] [reps]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1403_6015_b200 import inputs
import paper_1403_6015_b200.hodlr as hb
name = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
cfg = inputs.CONFIGS[name]
x = torch.from_numpy(inputs.points(cfg)).cuda(); y = torch.from_numpy(inputs.rhs(cfg)).cuda()
for _ in range(reps):
    h = hb.HODLR(x, cfg.kernel, cfg.theta, cfg.sigma2, cfg.leaf, cfg.eps)
    s, _ = h.factor_solve(y)
    ld = h.logdet()
    info = h.info(); h.close()
torch.cuda.synchronize()
print("logdet", ld, "kernel_ms", {k: round(v, 3) for k, v in info["kernel_ms"].items()})
