"""Scaling projection on ONE B200 (verdict r1 item 7): the sharded path's rank-0 critical path at
P = 2, 4, 8.  A recorded run executes all P virtual ranks (host threads, in-process transport) and keeps rank 0's
gathered exchange buffers; then rank 0 runs ALONE, each exchange replaying the recorded buffer with its own slot
live (hodlr_group_mode 2), and its device time is measured with CUDA events (median of reps, L2 flushed).  The
projection adds a modeled NVLink/NCCL allgather latency per exchange (15 us; 10-20 us each).  It is a
labelled projection, not a multi-GPU measurement.   python tools/project_scaling.py [cfg3] [out.json]"""
import json, os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1403_6015_b200 import inputs
import paper_1403_6015_b200.hodlr as hb
from paper_1403_6015_b200.dist import Group, Dist, run_virtual_ranks

name = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
cfg = inputs.CONFIGS[name]
x = torch.from_numpy(inputs.points(cfg)).cuda(); y = torch.from_numpy(inputs.rhs(cfg)).cuda()
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
EXCH_US = 15.0


def step(d):
    h = hb.HODLR(x, cfg.kernel, cfg.theta, cfg.sigma2, cfg.leaf, cfg.eps, dist=d)
    s, _ = h.factor_solve(y)
    ld = h.logdet(); info = h.info(); h.close()
    return ld, info


def timed(fn, reps=5):
    ts, out = [], None
    for _ in range(reps):
        flush.zero_(); torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); out = fn(); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts), out


res = {"config": name, "n": cfg.n, "model": f"rank-0 solo replay + {EXCH_US:g} us per allgather (modeled)", "P": {}}
step(None); step(None)
t1, (ld1, info1) = timed(lambda: step(None))
res["P"]["1"] = {"ms": t1, "points_per_s": cfg.n / (t1 * 1e-3), "aca_ms": info1["kernel_ms"]["aca"]}
print(f"P=1: {t1:.3f} ms", flush=True)
for P in (2, 4, 8):
    g = Group(P)
    g.mode(1)
    s = torch.cuda.Stream()

    def fn(r, d):
        with torch.cuda.stream(s if r == 0 else torch.cuda.Stream()):
            return step(d)
    rec = run_virtual_ranks(P, fn, g)
    nex = None
    ld_ref = rec[0][0]

    def solo():
        g.mode(2)
        return step(Dist(0, P, group=g))
    solo(); solo()
    tP, (ldP, infoP) = timed(solo)
    assert ldP == ld_ref, (ldP, ld_ref)
    g.close()
    nex = 4                    # exchanges per step with y fused: ranks (build), depth-t Pi, log det (factor), solution
    proj = tP + nex * EXCH_US * 1e-3
    res["P"][str(P)] = {"rank0_solo_ms": tP, "exchanges": nex, "projected_ms": proj,
                        "projected_points_per_s": cfg.n / (proj * 1e-3), "projected_speedup": t1 / proj,
                        "aca_ms_rank0": infoP["kernel_ms"]["aca"], "coupling_tree_ms_rank0": infoP["kernel_ms"]["coupling_tree"],
                        "leaf_factor_ms_rank0": infoP["kernel_ms"]["leaf_factor"], "logdet_equal_to_recorded": True}
    print(f"P={P}: rank-0 solo {tP:.3f} ms, projected {proj:.3f} ms ({t1 / proj:.2f}x), ACA {infoP['kernel_ms']['aca']:.3f} ms",
          flush=True)
out = sys.argv[2] if len(sys.argv) > 2 else None
if out:
    json.dump(res, open(out, "w"), indent=1)
