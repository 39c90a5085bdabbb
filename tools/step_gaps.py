"""Where the bench step's device time goes between the API calls: CUDA events around hodlr_build and
hodlr_factor_solve (device spans) against the per-family kernel event times inside them.  python tools/step_gaps.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1403_6015_b200 import inputs
import paper_1403_6015_b200.hodlr as hb
cfg = inputs.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg3"]
x = torch.from_numpy(inputs.points(cfg)).cuda(); y = torch.from_numpy(inputs.rhs(cfg)).cuda()
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
st = torch.cuda.current_stream()
for i in range(8):
    flush.zero_()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    ev[0].record(st)
    h = hb.HODLR(x, cfg.kernel, cfg.theta, cfg.sigma2, cfg.leaf, cfg.eps)
    ev[1].record(st)
    s, q = h.factor_solve(y)
    ev[2].record(st)
    ld = h.logdet()
    ev[3].record(st)
    info = h.info(); h.close()
    torch.cuda.synchronize()
    k = info["kernel_ms"]
    if i >= 3:
        print(f"build span {ev[0].elapsed_time(ev[1]):.3f} (sort {k['sort']:.3f} aca {k['aca']:.3f} chol {k['leaf_chol']:.3f}) "
              f"factor_solve span {ev[1].elapsed_time(ev[2]):.3f} (zsyrk {k['leaf_factor']:.3f} tree {k['coupling_tree']:.3f} "
              f"solve {k['solve']:.3f}) logdet {ev[2].elapsed_time(ev[3]):.3f} total {ev[0].elapsed_time(ev[3]):.3f}")
