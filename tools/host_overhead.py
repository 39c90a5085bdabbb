"""Wall-clock per API call vs device time (test tooling).  python tools/host_overhead.py [cfg]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1403_6015_b200 import inputs
import paper_1403_6015_b200.hodlr as hb
cfg = inputs.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg3"]
x = torch.from_numpy(inputs.points(cfg)).cuda(); y = torch.from_numpy(inputs.rhs(cfg)).cuda()
for rep in range(4):
    torch.cuda.synchronize()
    t0 = time.perf_counter(); h = hb.HODLR(x, cfg.kernel, cfg.theta, cfg.sigma2, cfg.leaf, cfg.eps)
    t1 = time.perf_counter(); h.factor()
    t2 = time.perf_counter(); ld = h.logdet()
    t3 = time.perf_counter(); s = h.solve(y)
    t4 = time.perf_counter(); info = h.info(); h.close(); torch.cuda.synchronize()
    t5 = time.perf_counter()
    print(f"wall ms: build {1e3*(t1-t0):.2f} factor {1e3*(t2-t1):.2f} logdet {1e3*(t3-t2):.2f} solve {1e3*(t4-t3):.2f} "
          f"close {1e3*(t5-t4):.2f} total {1e3*(t5-t0):.2f} | device t_build {1e3*info['t_build']:.2f} "
          f"t_factor {1e3*info['t_factor']:.2f} t_solve {1e3*info['t_solve']:.2f}", flush=True)
