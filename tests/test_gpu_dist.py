"""Subtree sharding on one B200 (-m gpu): P virtual ranks (host threads, in-process transport) run the
sharded path -- own subtree ACA/leaves/tree levels, redundant top levels, allgather of the depth-log2(P)
projected Gram matrices, log det partials, solve projections and solution slices -- and must reproduce the
one-GPU factorization (same kernels on the same blocks: only the log det summation order differs) and the
oracle."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import OracleHODLR  # noqa: E402
from paper_1403_6015_b200 import inputs  # noqa: E402


@pytest.fixture(scope="module")
def hb():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1403_6015_b200.hodlr as hb
    hb.load()
    return hb


def sharded(hb, P, x, y, kernel, theta, s2, leaf, eps):
    from paper_1403_6015_b200.dist import run_virtual_ranks
    xd = torch.from_numpy(x).cuda(); yd = torch.from_numpy(y).cuda()
    torch.cuda.synchronize()

    def fn(r, d):
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            g = hb.HODLR(xd, kernel, theta, s2, leaf, eps, dist=d).factor()
            out = (g.logdet(), g.solve(yd).cpu().numpy(), g.gp_loglik(yd), g.info())
            g.close()
        return out
    return run_virtual_ranks(P, fn)


CASES = [("cfg1", 2048, 2), ("cfg1", 2048, 8), ("cfg3", 1 << 16, 2), ("cfg3", 1 << 16, 8), ("cfg2", 65536, 4),
         ("cfg5", 1 << 15, 4)]


@pytest.mark.parametrize("name,n,P", CASES, ids=[f"{a}-{b}-P{c}" for a, b, c in CASES])
def test_virtual_ranks_match_one_gpu(hb, name, n, P):
    cfg = inputs.scaled(inputs.CONFIGS[name], n)
    x = inputs.points(cfg); y = inputs.rhs(cfg)
    g = hb.HODLR(torch.from_numpy(x).cuda(), cfg.kernel, cfg.theta, cfg.sigma2, cfg.leaf, 1e-12).factor()
    ld1 = g.logdet(); x1 = g.solve(torch.from_numpy(y).cuda()).cpu().numpy(); ll1 = g.gp_loglik(torch.from_numpy(y).cuda())
    res = sharded(hb, P, x, y, cfg.kernel, cfg.theta, cfg.sigma2, cfg.leaf, 1e-12)
    for r, (ld, xs, ll, info) in enumerate(res):
        assert info["rank"] == r and info["nranks"] == P and info["split_depth"] == P.bit_length() - 1
        assert abs(ld - ld1) <= 1e-13 * abs(ld1), (r, ld, ld1)
        assert np.linalg.norm(xs - x1) <= 1e-13 * np.linalg.norm(x1), (r, np.linalg.norm(xs - x1) / np.linalg.norm(x1))
        assert abs(ll - ll1) <= 1e-13 * (abs(ll1) + abs(ld1))
    print(f"[sharded] {name} n={n} P={P}: logdet rel {abs(res[0][0] - ld1) / abs(ld1):.1e} "
          f"solve rel {np.linalg.norm(res[0][1] - x1) / np.linalg.norm(x1):.1e}")


def test_virtual_ranks_match_oracle(hb):
    cfg = inputs.scaled(inputs.CONFIGS["cfg3"], 1 << 14)
    x = inputs.points(cfg); y = inputs.rhs(cfg)
    o = OracleHODLR(x, cfg.kernel, cfg.theta, cfg.sigma2, cfg.leaf, 1e-12).factor()
    ld_o = o.logdet(); x_o = o.solve(y)
    for ld, xs, ll, _ in sharded(hb, 4, x, y, cfg.kernel, cfg.theta, cfg.sigma2, cfg.leaf, 1e-12):
        assert abs(ld - ld_o) <= 1e-9 * abs(ld_o)
        assert np.linalg.norm(xs - x_o) <= 1e-9 * np.linalg.norm(x_o)


def test_sharded_errors(hb):
    from paper_1403_6015_b200.dist import run_virtual_ranks
    xd = torch.linspace(0, 1, 256, dtype=torch.float64, device="cuda")

    def fn(r, d):
        try:
            hb.HODLR(xd, 0, (1.0, 0.1), 1e-2, 64, 1e-12, dist=d)     # kappa = 2 < log2(8)
        except hb.HodlrError as e:
            return e.status
        return "OK"
    assert run_virtual_ranks(8, fn) == ["EINVAL"] * 8


def test_loglik_sweep_matches_single_settings(hb):
    """Config 4 shape: several (ell, sigma2) settings through gp_loglik_sweep (batched handles, and 4 virtual
    ranks splitting the settings) equal the one-setting path and the oracle."""
    from paper_1403_6015_b200.dist import run_virtual_ranks
    cfg = inputs.CONFIGS["cfg4"]
    ell, s2 = inputs.sweep_settings(cfg)
    c = inputs.scaled(cfg, 1 << 13)
    x = inputs.points(c); y = inputs.rhs(c)
    ks = [0, 5, 17, 40, 63]
    th = np.array([[cfg.a, ell[k]] for k in ks]); sg = np.array([s2[k] for k in ks])
    xd = torch.from_numpy(x).cuda(); yd = torch.from_numpy(y).cuda()
    vals = hb.gp_loglik_sweep(xd, yd, cfg.kernel, th, sg, cfg.leaf, 1e-12, workers=3)
    import math
    for j, k in enumerate(ks):
        g = hb.HODLR(xd, cfg.kernel, (cfg.a, ell[k]), s2[k], cfg.leaf, 1e-12)
        _, quad = g.factor_solve(yd, solve=False)         # y fused into the factorization, one setting
        one = -0.5 * quad - 0.5 * g.logdet() - 0.5 * c.n * math.log(2 * math.pi)
        assert abs(vals[j] - one) <= 1e-12 * abs(one)         # the sweep batches: summation order only
        two = hb.HODLR(xd, cfg.kernel, (cfg.a, ell[k]), s2[k], cfg.leaf, 1e-12).factor().gp_loglik(yd)
        assert abs(two - one) <= 1e-12 * abs(one)             # the unfused factor + loglik path
        o = OracleHODLR(x, cfg.kernel, (cfg.a, ell[k]), s2[k], cfg.leaf, 1e-12).factor()
        assert abs(vals[j] - o.gp_loglik(y)) <= 1e-9 * abs(o.gp_loglik(y)) + 1e-9 * abs(o.logdet())
    res = run_virtual_ranks(4, lambda r, d: hb.gp_loglik_sweep(xd, yd, cfg.kernel, th, sg, cfg.leaf, 1e-12, dist=d))
    for v in res:
        np.testing.assert_allclose(v, vals, rtol=1e-12, atol=0)   # (ranks batch different subsets)


@pytest.mark.parametrize("flag", ["HODLR_CHOL_AFTER_ACA"])
def test_alternate_paths_match(hb, flag):
    """The opt-in variants (fused leaf pairs + deepest tree level; Cholesky after the ACA) give the same
    factorization as the default path: run in a subprocess with the switch set."""
    import subprocess, sys, os, json
    code = ("import json,sys,torch; sys.path.insert(0,'.');"
            "from paper_1403_6015_b200 import inputs; import paper_1403_6015_b200.hodlr as hb;"
            "cfg=inputs.scaled(inputs.CONFIGS['cfg3'],1<<15); x=inputs.points(cfg); y=inputs.rhs(cfg);"
            "g=hb.HODLR(torch.from_numpy(x).cuda(),cfg.kernel,cfg.theta,cfg.sigma2,cfg.leaf,1e-12).factor();"
            "print(json.dumps([g.logdet(), g.solve(torch.from_numpy(y).cuda()).cpu().tolist()]))")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = []
    for env in ({}, {flag: "1"}):
        r = subprocess.run([sys.executable, "-c", code], cwd=root, env={**os.environ, **env}, capture_output=True,
                           text=True, timeout=300)
        assert r.returncode == 0, r.stderr[-2000:]
        outs.append(json.loads(r.stdout.strip().splitlines()[-1]))
    (ld0, x0), (ld1, x1) = outs
    x0 = np.array(x0); x1 = np.array(x1)
    assert abs(ld1 - ld0) <= 1e-12 * abs(ld0)
    assert np.linalg.norm(x1 - x0) <= 1e-10 * np.linalg.norm(x0)


@pytest.mark.parametrize("name,n,P", [("cfg1", 2048, 4), ("cfg3", 1 << 16, 8)])
def test_virtual_ranks_factor_solve(hb, name, n, P):
    """Sharded hodlr_factor_solve (y fused into the factorization; only the down passes after it) reproduces the
    one-GPU fused result and returns the full solution on every rank."""
    from paper_1403_6015_b200.dist import run_virtual_ranks
    cfg = inputs.scaled(inputs.CONFIGS[name], n)
    x = inputs.points(cfg); y = inputs.rhs(cfg)
    xd = torch.from_numpy(x).cuda(); yd = torch.from_numpy(y).cuda()
    g = hb.HODLR(xd, cfg.kernel, cfg.theta, cfg.sigma2, cfg.leaf, 1e-12)
    x1, q1 = g.factor_solve(yd); x1 = x1.cpu().numpy(); ld1 = g.logdet()
    torch.cuda.synchronize()

    def fn(r, d):
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            h = hb.HODLR(xd, cfg.kernel, cfg.theta, cfg.sigma2, cfg.leaf, 1e-12, dist=d)
            xs, q = h.factor_solve(yd)
            out = (h.logdet(), xs.cpu().numpy(), q)
            h.close()
        return out
    for ld, xs, q in run_virtual_ranks(P, fn):
        assert abs(ld - ld1) <= 1e-13 * abs(ld1)
        assert abs(q - q1) <= 1e-12 * abs(q1)
        assert np.linalg.norm(xs - x1) <= 1e-12 * np.linalg.norm(x1)


def test_group_record_replay(hb):
    """hodlr_group_mode (the scaling projection of tools/project_scaling.py): rank 0 replayed alone against the
    recorded exchanges of a full P-rank run computes the same log det and solution as in that run."""
    from paper_1403_6015_b200.dist import Group, Dist, run_virtual_ranks
    cfg = inputs.scaled(inputs.CONFIGS["cfg3"], 1 << 15)
    xd = torch.from_numpy(inputs.points(cfg)).cuda(); yd = torch.from_numpy(inputs.rhs(cfg)).cuda()

    def step(d):
        h = hb.HODLR(xd, cfg.kernel, cfg.theta, cfg.sigma2, cfg.leaf, 1e-12, dist=d)
        s, q = h.factor_solve(yd)
        out = (h.logdet(), q, s.cpu().numpy())
        h.close()
        return out
    g = Group(4)
    g.mode(1)
    rec = run_virtual_ranks(4, lambda r, d: step(d), g)
    g.mode(2)
    ld, q, s = step(Dist(0, 4, group=g))
    g.close()
    assert ld == rec[0][0] and q == rec[0][1]
    np.testing.assert_array_equal(s, rec[0][2])
