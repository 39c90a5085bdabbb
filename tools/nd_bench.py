"""NEXT-3 measurement: one B200, d-dimensional workloads (inputs.ND_CONFIGS, Table II's uniform cube
shape), step = hodlr_build_nd + hodlr_factor_solve + hodlr_logdet with the inputs resident in HBM, L2 flushed
between steps (512 MB write, untimed), CUDA events, median of K steps after W warm-ups; per step the SURVEY App. B
combined roofline with this run's ranks (the ACA and leaf entries read d coordinates and evaluate a d-term distance:
8 n d bytes for the points, 3 (d - 1) more flops per entry).  python tools/nd_bench.py [out.json]"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1403_6015_b200 import inputs
import paper_1403_6015_b200.hodlr as hb
import bench

PEAKS = bench.load_peaks()
F_PEAK = 37.13e12                                        # measured DMMA peak (profiles/fp64_peak_r01.json)
B_PEAK = float(PEAKS.get("hbm_gbs", 6532.9)) * 1e9 if isinstance(PEAKS, dict) else 6532.9e9
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")


def t_roof_nd(info, n, p, d):
    ph = bench.app_b(info, n, p)
    K = sum(info["max_rank_by_depth"])
    f, b = ph["B_aca"]
    ph["B_aca"] = (f + 3 * (d - 1) * n * K, b + 8 * n * (d - 1))
    f, b = ph["C_leaf_chol"]
    ph["C_leaf_chol"] = (f + 3 * (d - 1) * n * p / 2, b + 8 * n * (d - 1))
    return 1e3 * sum(max(f / F_PEAK, b / B_PEAK) for f, b in ph.values())


def run(name, n, warm=3, reps=7):
    d, half, kernel, theta, s2, leaf, eps = inputs.ND_CONFIGS[name]
    x, y = inputs.points_nd(n, d, seed=2, half=half)
    xd = torch.from_numpy(x).cuda(); yd = torch.from_numpy(y).cuda()

    def step():
        h = hb.HODLR(xd, kernel, theta, s2, leaf, eps)
        _, quad = h.factor_solve(yd)
        ld = h.logdet(); info = h.info(); h.close()
        return ld, quad, info
    for _ in range(warm):
        step()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        flush.zero_()
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); ld, quad, info = step(); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ms = sorted(ts)[len(ts) // 2]
    tr = t_roof_nd(info, n, leaf, d)
    return {"workload": name, "d": d, "n": n, "kernel": kernel, "theta": theta, "sigma2": s2, "leaf": leaf, "eps": eps,
            "ms_per_step": ms, "points_per_s": n / (ms * 1e-3), "samples_ms": [round(t, 3) for t in ts],
            "logdet": ld, "K": info["K"], "kappa": info["kappa"],
            "ranks_by_depth": info["max_rank_by_depth"], "t_roof_ms_app_b": tr, "roofline_frac": tr / ms,
            "kernel_family_ms": {k: round(v, 3) for k, v in info["kernel_ms"].items() if not k.startswith("unused")},
            "gpu_launches_build": None}


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "once":     # profiling: python tools/nd_bench.py once nd2 20
        print(json.dumps(run(sys.argv[2], 1 << int(sys.argv[3]), warm=1, reps=1)))
        sys.exit(0)
    res = {"device": torch.cuda.get_device_name(0), "l2": "flushed between timed steps (512 MB write, untimed)",
           "runs": []}
    for name, n in (("nd2", 1 << 16), ("nd2", 1 << 18), ("nd2", 1 << 20), ("nd3", 1 << 16), ("nd3", 1 << 18)):
        try:
            r = run(name, n)
        except Exception as e:                          # a size whose coupling systems do not fit is reported
            r = {"workload": name, "n": n, "error": str(e)}
        res["runs"].append(r)
        print(json.dumps(r), flush=True)
    if len(sys.argv) > 1:
        json.dump(res, open(sys.argv[1], "w"), indent=1)
