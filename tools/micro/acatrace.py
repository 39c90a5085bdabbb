import sys, ctypes as C, numpy as np, torch
sys.path.insert(0, '.')
from paper_1403_6015_b200 import inputs
import paper_1403_6015_b200.hodlr as hb
cfg = inputs.CONFIGS['cfg3']; x = inputs.points(cfg)
g = hb.HODLR(torch.from_numpy(x).cuda(), cfg.kernel, cfg.theta, cfg.sigma2, cfg.leaf, 1e-12)
torch.cuda.synchronize()
print("gpu rank block 15:", g.tree()[2][15], flush=True)
lib = C.CDLL('oracle/liboracle_trace.so')
lib.oracle_build.argtypes = [C.c_void_p, C.c_int64, C.c_int, C.c_void_p, C.c_double, C.c_int, C.c_double, C.c_int, C.c_void_p]
th = np.array([cfg.a, cfg.ell, 0.0]); h = C.c_void_p(0)
print("oracle build", lib.oracle_build(x.ctypes.data, x.size, 0, th.ctypes.data, cfg.sigma2, cfg.leaf, 1e-12, 0, C.byref(h)), flush=True)
