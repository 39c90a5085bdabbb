"""One build + factor of the paper's Table II 1-D shape with leaf 128 (leaves of 244 / 245 points: k_leaf_factor),
for ncu captures of the scalar leaf path.  python tools/prof_leaf_fallback.py [n]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1403_6015_b200.hodlr as hb
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1000000
rng = np.random.default_rng(7)
x = rng.uniform(-3, 3, n)
h = hb.HODLR(torch.from_numpy(x).cuda(), 0, (1.0, 2 ** -0.5), 2.0, 128, 1e-12).factor()
print(h.logdet(), h.info()["kernel_ms"])
h.close()
