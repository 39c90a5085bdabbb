"""Probe of bench.py's end-to-end step (host buffers in, solution out): per-step device time and host time per API
call, to find stalls.  python tools/e2e_probe.py [steps]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1403_6015_b200 import inputs
import paper_1403_6015_b200.hodlr as hb
cfg = inputs.CONFIGS["cfg3"]
steps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
x = inputs.points(cfg); y = inputs.rhs(cfg)
xh = torch.from_numpy(x).pin_memory(); yh = torch.from_numpy(y).pin_memory()
xd = torch.empty(cfg.n, dtype=torch.float64, device="cuda"); yd = torch.empty_like(xd)
sol_h = torch.empty(cfg.n, dtype=torch.float64).pin_memory()
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
stream = torch.cuda.current_stream(); ys = torch.cuda.Stream(); ev_y = torch.cuda.Event()
xd0 = torch.from_numpy(x).cuda(); yd0 = torch.from_numpy(y).cuda()
for i in range(8):          # the bench's device-resident warm-up + timed steps first
    flush.zero_()
    h = hb.HODLR(xd0, cfg.kernel, cfg.theta, cfg.sigma2, cfg.leaf, cfg.eps); s, _ = h.factor_solve(yd0); h.logdet(); h.close()
torch.cuda.synchronize()
for i in range(steps):
    flush.zero_()
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record(stream)
    t = [time.perf_counter()]
    xd.copy_(xh, non_blocking=True)
    ys.wait_stream(stream)
    with torch.cuda.stream(ys):
        yd.copy_(yh, non_blocking=True); ev_y.record(ys)
    h = hb.HODLR(xd, cfg.kernel, cfg.theta, cfg.sigma2, cfg.leaf, cfg.eps); t.append(time.perf_counter())
    stream.wait_event(ev_y)
    s, _ = h.factor_solve(yd); t.append(time.perf_counter())
    ld = h.logdet()
    sol_h.copy_(s, non_blocking=True)
    h.close(); t.append(time.perf_counter())
    b.record(stream); torch.cuda.synchronize(); t.append(time.perf_counter())
    d = [1e3 * (t[k + 1] - t[k]) for k in range(len(t) - 1)]
    print(f"step {i}: device {a.elapsed_time(b):7.3f} ms; host build {d[0]:.3f} factor_solve {d[1]:.3f} "
          f"logdet+copy+free {d[2]:.3f} tail {d[3]:.3f}", flush=True)
