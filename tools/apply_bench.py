"""Forward apply (hodlr_apply) timing on a BASELINE config: device-resident x, CUDA events, L2 flushed between
calls.  python tools/apply_bench.py [cfg3] [reps]"""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1403_6015_b200 import inputs
import paper_1403_6015_b200.hodlr as hb
name = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
cfg = inputs.CONFIGS[name]
x = torch.from_numpy(inputs.points(cfg)).cuda(); v = torch.from_numpy(inputs.rhs(cfg)).cuda()
h = hb.HODLR(x, cfg.kernel, cfg.theta, cfg.sigma2, cfg.leaf, cfg.eps)
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
for _ in range(3):
    h.apply(v)
torch.cuda.synchronize()
ts = []
for _ in range(reps):
    flush.zero_()
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record(); y = h.apply(v); b.record(); torch.cuda.synchronize()
    ts.append(a.elapsed_time(b))
info = h.info()
K = info["K"]; n = cfg.n
byts = 2 * 8 * n * K + 3 * 8 * n            # panel read twice (E^T x, E w) + x, y, ys
ms = sorted(ts)[len(ts) // 2]
print(json.dumps({"config": name, "n": n, "K": K, "apply_ms_median": ms, "points_per_s": n / (ms * 1e-3),
                  "panel_bytes": byts, "achieved_GBps": byts / (ms * 1e-3) / 1e9,
                  "leaf_entries": int(n * cfg.leaf)}))
