"""The paper's Table II 1-D row at n = 10^6 (C = 2 I + exp(-|r_i - r_j|^2), r_i ~ U[-3, 3], PAPER.md:1302-1308, 1345;
eps = 1e-12) on one B200: build + factor_solve + logdet with x, y resident, CUDA events, L2 flushed, median of 5 after
2 warm-ups; leaf 128 (leaves of 244 / 245 points: the scalar leaf path) and leaf 64 (leaves of 122 / 123: DMMA).
python tools/paper_shape.py [out.json]"""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1403_6015_b200.hodlr as hb
n = 1000000
rng = np.random.default_rng(7)
x = rng.uniform(-3, 3, n); y = rng.standard_normal(n)
xd = torch.from_numpy(x).cuda(); yd = torch.from_numpy(y).cuda()
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
res = []
for leaf in (128, 64):
    ts = []
    for rep in range(7):
        flush.zero_()
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record()
        h = hb.HODLR(xd, 0, (1.0, 2 ** -0.5), 2.0, leaf, 1e-12)
        s, q = h.factor_solve(yd); ld = h.logdet(); info = h.info(); h.close()
        b.record(); torch.cuda.synchronize()
        if rep >= 2:
            ts.append(a.elapsed_time(b))
    r = {"n": n, "leaf": leaf, "ms_per_step": sorted(ts)[len(ts) // 2], "samples_ms": [round(t, 3) for t in ts],
         "points_per_s": n / (sorted(ts)[len(ts) // 2] * 1e-3), "logdet": ld, "kappa": info["kappa"], "K": info["K"],
         "leaf_min": info.get("leaf_min"), "leaf_max": info.get("leaf_max"),
         "ranks_by_depth": info["max_rank_by_depth"],
         "kernel_family_ms": {k: round(v, 3) for k, v in info["kernel_ms"].items() if not k.startswith("unused")}}
    res.append(r)
    print(json.dumps(r), flush=True)
if len(sys.argv) > 1:
    json.dump(res, open(sys.argv[1], "w"), indent=1)
