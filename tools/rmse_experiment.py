"""sec. 5.6 regression experiment on the GPU path: |RMSE(HODLR, eps) - RMSE(dense)| for the
synthetic model y = sin 2x + e^x / 8 + N(0, 1), 1024 points in (-3, 3), k = exp(-(x - x')^2), sigma_eps = 1,
p_max = 20.  Writes one JSON object.  python tools/rmse_experiment.py [out.json]"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1403_6015_b200 import inputs
import paper_1403_6015_b200.hodlr as hb
x, y = inputs.rmse_model()
theta, s2, leaf = (1.0, 1.0 / np.sqrt(2.0)), 1.0, 20
d = x[:, None] - x[None, :]
K = np.exp(-d * d)
rmse_exact = float(np.linalg.norm(y - K @ np.linalg.solve(K + s2 * np.eye(x.size), y)) / np.sqrt(x.size))
xd = torch.from_numpy(x).cuda(); yd = torch.from_numpy(y).cuda()
rows = []
for eps in [10.0 ** -k for k in range(1, 14)]:
    g = hb.HODLR(xd, hb.HODLR_SE, theta, s2, leaf, eps).factor()
    yhat = (yd - s2 * g.solve(yd)).cpu().numpy()
    rmse = float(np.linalg.norm(y - yhat) / np.sqrt(x.size))
    rows.append({"eps": eps, "rmse": rmse, "abs_diff": abs(rmse - rmse_exact),
                 "max_rank": int(max(g.info()["max_rank_by_depth"][:g.info()["kappa"]] or [0]))})
    g.close()
out = {"experiment": "sec. 5.6 regression (PAPER.md:1656-1705), synthetic, seed 56", "n": int(x.size),
       "rmse_dense": rmse_exact, "paper_rmse_dense_for_its_own_draw": 0.9969571605921435, "rows": rows}
s = json.dumps(out, indent=1)
print(s)
if len(sys.argv) > 1:
    open(sys.argv[1], "w").write(s)
