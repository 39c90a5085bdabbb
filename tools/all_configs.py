"""One B200: build + factor + logdet + solve timed on every BASELINE config (device-resident inputs, CUDA events,
L2 flushed between steps, median of K steps after W warm-ups), the config-4 sweep through gp_loglik_sweep, and the
forward apply / prediction at config 3.  Writes one JSON object.  python tools/all_configs.py [out.json]"""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1403_6015_b200 import inputs
import paper_1403_6015_b200.hodlr as hb

flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
import bench                                             # App. B counts and the measured peaks
PEAKS = bench.load_peaks()
F_PEAK = 37.13e12                                        # measured DMMA peak (profiles/fp64_peak_r01.json)
B_PEAK = float(PEAKS.get("hbm_gbs", 6532.9)) * 1e9 if isinstance(PEAKS, dict) else 6532.9e9


def t_roof(info, n, p, ranks=None):
    """SURVEY App. B combined roofline sum_phase max(F / F_peak, B / B_peak) in ms, with this run's ranks."""
    inf = dict(info)
    if ranks is not None:
        inf["max_rank_by_depth"] = ranks
    ph = bench.app_b(inf, n, p)
    return 1e3 * sum(max(f / F_PEAK, b / B_PEAK) for f, b in ph.values())


def timed(fn, warm=2, reps=5):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        flush.zero_()
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); out = fn(); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return sorted(ts)[len(ts) // 2], out


res = {"device": torch.cuda.get_device_name(0), "configs": {}}
for name in ("cfg1", "cfg2", "cfg3", "cfg5"):
    cfg = inputs.CONFIGS[name]
    x = torch.from_numpy(inputs.points(cfg)).cuda(); y = torch.from_numpy(inputs.rhs(cfg)).cuda()

    def step():
        h = hb.HODLR(x, cfg.kernel, cfg.theta, cfg.sigma2, cfg.leaf, cfg.eps)
        s, _ = h.factor_solve(y)
        ld = h.logdet(); info = h.info(); h.close()
        return ld, info
    ms, (ld, info) = timed(step, reps=3 if cfg.n > (1 << 21) else 5)
    tr = t_roof(info, cfg.n, cfg.leaf)
    res["configs"][name] = {"n": cfg.n, "ms_per_step": ms, "points_per_s": cfg.n / (ms * 1e-3), "logdet": ld,
                            "t_roof_ms_app_b": tr, "roofline_frac": tr / ms,
                            "K": info["K"], "kappa": info["kappa"],
                            "kernel_family_ms": {k: round(v, 3) for k, v in info["kernel_ms"].items() if not k.startswith("unused")}}
    print(name, json.dumps(res["configs"][name]), flush=True)
cfg = inputs.CONFIGS["cfg4"]
ell, s2 = inputs.sweep_settings(cfg)
x = torch.from_numpy(inputs.points(cfg)).cuda(); y = torch.from_numpy(inputs.rhs(cfg)).cuda()
th = np.stack([np.full(cfg.sweep, cfg.a), ell], 1)
hb.gp_loglik_sweep(x, y, cfg.kernel, th, s2, cfg.leaf, cfg.eps)          # warm-up (allocations, plans)
ts = []
for _ in range(5):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    v = hb.gp_loglik_sweep(x, y, cfg.kernel, th, s2, cfg.leaf, cfg.eps)
    torch.cuda.synchronize(); ts.append(1e3 * (time.perf_counter() - t0))
t = float(np.median(ts)) / 1e3
g = hb.HODLRBatch(x, cfg.kernel, th, s2, cfg.leaf, cfg.eps)          # ranks of the batched handle (per setting below
g.factor_solve(y.repeat(cfg.sweep), solve=False)                   # the problem-coupling depths)
binfo = g.info(); g.close()
tsb = cfg.sweep.bit_length() - 1
tr4 = cfg.sweep * t_roof(binfo, cfg.n, cfg.leaf, ranks=list(binfo["max_rank_by_depth"])[tsb:])
res["configs"]["cfg4"] = {"n": cfg.n, "settings": cfg.sweep, "ms_per_sweep_wall": 1e3 * t, "samples_ms": ts,
                          "t_roof_ms_app_b": tr4, "roofline_frac": tr4 / (1e3 * t),
                          "path": "batched handles (hodlr_build_batch, 64 settings in one handle)",
                          "settings_per_s": cfg.sweep / t, "loglik_min": float(v.min()), "loglik_max": float(v.max())}
print("cfg4", json.dumps(res["configs"]["cfg4"]), flush=True)
cfg = inputs.CONFIGS["cfg3"]
x = torch.from_numpy(inputs.points(cfg)).cuda(); y = torch.from_numpy(inputs.rhs(cfg)).cuda()
h = hb.HODLR(x, cfg.kernel, cfg.theta, cfg.sigma2, cfg.leaf, cfg.eps).factor()
ms_apply, _ = timed(lambda: h.apply(y))
xt = torch.linspace(cfg.lo, cfg.hi, 1024, dtype=torch.float64, device="cuda")
ms_mean, _ = timed(lambda: h.predict(y, xt, variance=False), reps=3)
xt32 = xt[:32].contiguous()
ms_var, _ = timed(lambda: h.predict(y, xt32, variance=True), warm=1, reps=3)
res["cfg3_next1"] = {"apply_ms": ms_apply, "predict_mean_1024_test_points_ms": ms_mean,
                     "predict_mean_and_variance_32_test_points_ms": ms_var}
print("cfg3 next-1", json.dumps(res["cfg3_next1"]), flush=True)
s = json.dumps(res, indent=1)
if len(sys.argv) > 1:
    open(sys.argv[1], "w").write(s)
