"""Small end-to-end run for compute-sanitizer (memcheck / racecheck / synccheck): config 1 and a config-2-shaped
problem through build, factor, factor_solve, solve, gp_loglik, apply, predict and the sharded path (2 virtual ranks).
python tools/sanitize_run.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1403_6015_b200 import inputs
import paper_1403_6015_b200.hodlr as hb
from paper_1403_6015_b200.dist import run_virtual_ranks
for name, n in (("cfg1", 2048), ("cfg2", 8192), ("cfg3", 16384)):
    cfg = inputs.scaled(inputs.CONFIGS[name], n)
    x = torch.from_numpy(inputs.points(cfg, sort=False)).cuda(); y = torch.from_numpy(inputs.rhs(cfg)).cuda()
    g = hb.HODLR(x, cfg.kernel, cfg.theta, cfg.sigma2, cfg.leaf, 1e-12)
    s, q = g.factor_solve(y)
    s2 = g.solve(torch.stack([y, 2 * y], 1)); ll = g.gp_loglik(y); a = g.apply(y)
    m, v = g.predict(y, x[:40].contiguous() + 1e-3)
    g.close()
    g = hb.HODLR(x, cfg.kernel, cfg.theta, cfg.sigma2, cfg.leaf, 1e-12).factor()
    s3 = g.solve(y); g.close()
    res = run_virtual_ranks(2, lambda r, d: hb.HODLR(x, cfg.kernel, cfg.theta, cfg.sigma2, cfg.leaf, 1e-12,
                                                     dist=d).factor().logdet())
    torch.cuda.synchronize()
    print(name, n, float(q), float(ll), float((s - s3).abs().max()), res[0] == res[1], flush=True)
