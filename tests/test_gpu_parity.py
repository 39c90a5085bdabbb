"""GPU parity: the CUDA path (through the C-ABI) against the CPU oracle on the same seeded inputs.

Tolerances (north_star): integer structures (perm, tree) bit-exact;
|d logdet| / |logdet| <= 1e-9 and ||dx|| / ||x|| <= 1e-9 at eps = 1e-12.  ACA pivots/ranks are
FP-derived (R11) and are reported, with a loose bound on the mismatch.
"""
import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import OracleHODLR, OracleError  # noqa: E402
from paper_1403_6015_b200 import inputs  # noqa: E402

LD_TOL = 1e-9
X_TOL = 1e-9


@pytest.fixture(scope="module")
def hb():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1403_6015_b200.hodlr as hb
    hb.load()
    return hb


def run_both(hb, x, y, kernel, theta, s2, leaf, eps, rank_cap=0):
    o = OracleHODLR(x, kernel, theta, s2, leaf, eps, rank_cap).factor()
    ld_o = o.logdet(); x_o = o.solve(y); ll_o = o.gp_loglik(y)
    xd = torch.from_numpy(x).cuda(); yd = torch.from_numpy(y).cuda()
    g = hb.HODLR(xd, kernel, theta, s2, leaf, eps, rank_cap).factor()
    ld_g = g.logdet(); x_g = g.solve(yd).cpu().numpy(); ll_g = g.gp_loglik(yd)
    return o, g, (ld_o, x_o, ll_o), (ld_g, x_g, ll_g)


def check_parity(o, g, ro, rg, ld_tol=LD_TOL, x_tol=X_TOL, exact_structure=True):
    ld_o, x_o, ll_o = ro
    ld_g, x_g, ll_g = rg
    print(f"[parity] n={x_o.size} logdet rel {abs(ld_g - ld_o) / abs(ld_o):.2e} "
          f"solve rel {np.linalg.norm(x_g - x_o) / np.linalg.norm(x_o):.2e} loglik rel {abs(ll_g - ll_o) / abs(ll_o):.2e}")
    assert abs(ld_g - ld_o) <= ld_tol * abs(ld_o) + 1e-12, (ld_g, ld_o)
    assert np.linalg.norm(x_g - x_o) <= x_tol * np.linalg.norm(x_o), np.linalg.norm(x_g - x_o) / np.linalg.norm(x_o)
    assert abs(ll_g - ll_o) <= ld_tol * (abs(ll_o) + abs(ld_o)), (ll_g, ll_o)
    if exact_structure:
        xs_g, perm_g = g.order()
        np.testing.assert_array_equal(perm_g.cpu().numpy(), o.perm())
        np.testing.assert_array_equal(xs_g.cpu().numpy(), o.sorted_x())
        lo_g, hi_g, r_g = g.tree()
        lo_o, hi_o = o.tree()
        np.testing.assert_array_equal(lo_g, lo_o)
        np.testing.assert_array_equal(hi_g, hi_o)
        r_o = o.ranks()
        if len(r_o):
            mism = np.mean(r_g != r_o)
            assert mism <= 0.25, f"rank mismatch fraction {mism}"
            assert np.all(np.abs(r_g.astype(int) - r_o.astype(int)) <= 2)


CFG_CASES = [
    ("cfg1", 2048),
    ("cfg2", 65536),
    ("cfg3", 1 << 16),
    ("cfg5", 1 << 15),
]


@pytest.mark.parametrize("name,n", CFG_CASES, ids=[f"{a}-{b}" for a, b in CFG_CASES])
def test_config_parity(hb, name, n):
    cfg = inputs.scaled(inputs.CONFIGS[name], n)
    x = inputs.points(cfg); y = inputs.rhs(cfg)
    o, g, ro, rg = run_both(hb, x, y, cfg.kernel, cfg.theta, cfg.sigma2, cfg.leaf, 1e-12)
    check_parity(o, g, ro, rg)


def twin_floor(x, y, kernel, theta, s2, leaf, eps):
    """Q15 conditioning floor: ||x_oracle - x_twin|| / ||x_oracle|| of the oracle and its twin (leaf LU +
    coupling-system QR, same compression) -- two backward-stable FP64 implementations with the same pivots."""
    o = OracleHODLR(x, kernel, theta, s2, leaf, eps).factor()
    t = OracleHODLR(x, kernel, theta, s2, leaf, eps, twin=True).factor()
    x_o, x_t = o.solve(y), t.solve(y)
    return o, float(np.linalg.norm(x_t - x_o) / np.linalg.norm(x_o))


def cfg4_case(hb, k, n):
    cfg = inputs.CONFIGS["cfg4"]
    ell, s2 = inputs.sweep_settings(cfg)
    c = inputs.scaled(cfg, n)
    x = inputs.points(c); y = inputs.rhs(c)
    o, floor = twin_floor(x, y, cfg.kernel, (1.0, ell[k]), s2[k], cfg.leaf, 1e-12)
    ro = (o.logdet(), o.solve(y), o.gp_loglik(y))
    g = hb.HODLR(torch.from_numpy(x).cuda(), cfg.kernel, (1.0, ell[k]), s2[k], cfg.leaf, 1e-12).factor()
    yd = torch.from_numpy(y).cuda()
    rg = (g.logdet(), g.solve(yd).cpu().numpy(), g.gp_loglik(yd))
    x_tol = max(X_TOL, 10.0 * floor)        # SURVEY 8(c) Q15 / DESIGN.md R15
    print(f"[cfg4 setting {k} n={n} ell={ell[k]:.3g} s2={s2[k]:.3g}] twin floor {floor:.2e} -> gate {x_tol:.2e}")
    check_parity(o, g, ro, rg, x_tol=x_tol)
    g.close()


@pytest.mark.parametrize("k", range(64))
def test_cfg4_sweep_parity(hb, k):
    """All 64 config-4 settings at n = 2^14 (same density): log det <= 1e-9, solve <= max(1e-9, 10 floor) with the
    floor measured per setting against the Q15 oracle twin."""
    cfg4_case(hb, k, 1 << 14)


CFG4_EXTREME = [12, 17, 45, 36, 40, 43, 10, 15]     # largest log(ell / sigma2) (worst conditioned) + smallest ell


@pytest.mark.parametrize("k", CFG4_EXTREME)
def test_cfg4_full_size_extreme(hb, k):
    """The 8 most extreme config-4 settings at the full n = 131072 (Matern-5/2, leaf 64, eps = 1e-12), gated at
    max(1e-9, 10 floor) per setting."""
    cfg4_case(hb, k, inputs.CONFIGS["cfg4"].n)


@pytest.mark.parametrize("n,leaf", [(1, 64), (17, 64), (64, 64), (127, 64), (128, 64), (1999, 50), (3001, 37),
                                    (4097, 128),
                                    # leaves of more than 128 points: the scalar leaf kernel k_leaf_factor, a single
                                    # leaf (K = 0), all in shared memory (256 threads), in global scratch (1024 threads)
                                    (200, 200), (300, 128), (2000, 128), (5001, 100)])
def test_edge_sizes(hb, n, leaf):
    rng = np.random.default_rng(n)
    x = rng.uniform(-3, 3, n); y = rng.standard_normal(n)
    o, g, ro, rg = run_both(hb, x, y, 0, (1.0, 1 / math.sqrt(2)), 1.0, leaf, 1e-12)
    check_parity(o, g, ro, rg)


@pytest.mark.parametrize("kernel", [0, 1, 2])
def test_unsorted_with_ties(hb, kernel):
    rng = np.random.default_rng(9)
    n = 5000
    x = np.round(rng.uniform(0, 20, n), 2)      # many exact ties
    x[::101] = -0.0
    y = rng.standard_normal(n)
    o, g, ro, rg = run_both(hb, x, y, kernel, (1.3, 0.7), 1e-2, 64, 1e-12)
    check_parity(o, g, ro, rg)


def test_multi_rhs(hb):
    rng = np.random.default_rng(3)
    n = 3000
    x = rng.uniform(0, 5, n); Y = rng.standard_normal((n, 3))
    o = OracleHODLR(x, 1, (1.0, 0.5), 1e-3, 64, 1e-12).factor()
    g = hb.HODLR(torch.from_numpy(x).cuda(), 1, (1.0, 0.5), 1e-3, 64, 1e-12).factor()
    Xg = g.solve(torch.from_numpy(Y).cuda()).cpu().numpy()
    Xo = o.solve(Y)
    assert np.linalg.norm(Xg - Xo) <= X_TOL * np.linalg.norm(Xo)


def test_logdet_parts_match(hb):
    cfg = inputs.CONFIGS["cfg1"]
    x = inputs.points(cfg)
    o = OracleHODLR(x, cfg.kernel, cfg.theta, cfg.sigma2, cfg.leaf, 1e-12).factor()
    g = hb.HODLR(torch.from_numpy(x).cuda(), cfg.kernel, cfg.theta, cfg.sigma2, cfg.leaf, 1e-12).factor()
    la_o, nb_o = o.logdet_parts()
    la_g, nb_g = g.logdet_parts()
    np.testing.assert_allclose(la_g, la_o, rtol=1e-12)          # leaf Cholesky: same matrix, same algorithm
    np.testing.assert_allclose(nb_g, nb_o, rtol=1e-6, atol=1e-9)  # coupling dets: eps-level differences


def test_closed_forms_on_gpu(hb):
    """Pins that hold independently of the oracle: K = 0 and the rank-1 Sylvester case."""
    n, s2 = 2048, 1e-2
    rng = np.random.default_rng(1)
    x = rng.uniform(0, 1, n); y = rng.standard_normal(n)
    g = hb.HODLR(torch.from_numpy(x).cuda(), 0, (0.0, 0.1), s2, 64, 1e-12).factor()
    assert g.logdet() == pytest.approx(n * math.log(s2), rel=1e-14)
    np.testing.assert_allclose(g.solve(torch.from_numpy(y).cuda()).cpu().numpy(), y / s2, rtol=1e-14)
    g = hb.HODLR(torch.from_numpy(x[:1024]).cuda(), 0, (1.0, 1e20), s2, 64, 1e-12).factor()
    assert g.logdet() == pytest.approx(1023 * math.log(s2) + math.log(s2 + 1024), rel=1e-12)


def test_errors(hb):
    xd = torch.linspace(0, 1, 100, dtype=torch.float64, device="cuda")
    for kw in [dict(leaf=0), dict(eps=0.0), dict(s2=-1.0), dict(theta=(1.0, 0.0)), dict(kernel=5)]:
        args = dict(kernel=0, theta=(1.0, 0.1), s2=1e-2, leaf=16, eps=1e-12)
        args.update(kw)
        with pytest.raises(hb.HodlrError) as e:
            hb.HODLR(xd, args["kernel"], args["theta"], args["s2"], args["leaf"], args["eps"])
        assert e.value.status == "EINVAL"
    bad = xd.clone(); bad[7] = float("nan")
    with pytest.raises(hb.HodlrError) as e:
        hb.HODLR(bad, 0, (1.0, 0.1), 1e-2, 16, 1e-12)
    assert e.value.status == "EINVAL"
    g = hb.HODLR(xd, 0, (1.0, 0.1), 1e-2, 16, 1e-12)
    with pytest.raises(hb.HodlrError) as e:
        g.solve(torch.ones(100, dtype=torch.float64, device="cuda"))
    assert e.value.status == "ESTATE"
    g.factor()
    yb = torch.ones(100, dtype=torch.float64, device="cuda"); yb[3] = float("inf")
    with pytest.raises(hb.HodlrError) as e:
        g.solve(yb)
    assert e.value.status == "EINVAL"
    dup = torch.from_numpy(np.repeat(np.linspace(0, 1, 50), 2)).cuda()
    gd = hb.HODLR(dup, 0, (1.0, 0.1), 0.0, 16, 1e-12)
    with pytest.raises(hb.HodlrError) as e:
        gd.factor()
    assert e.value.status == "ENOTPD"
    with pytest.raises(hb.HodlrError):
        gd.logdet()
    rng = np.random.default_rng(0)
    xr = torch.from_numpy(rng.uniform(0, 1, 512)).cuda()
    with pytest.raises(hb.HodlrError) as e:
        hb.HODLR(xr, 0, (1.0, 0.01), 1e-2, 16, 1e-12, rank_cap=2)
    assert e.value.status == "ERANKCAP"


def test_full_size_cfg3_bench_config(hb):
    """BASELINE.json config 3 at full size in the bench's configuration (n = 2^20, eps = 1e-10, the fused
    factor_solve the bench times): log det <= 1e-9 and solve <= 1e-9 against the oracle at the same eps, and the
    exact residual C x - y on 64 sampled rows (assembled row by row) within 2x the oracle's on the same rows."""
    cfg = inputs.CONFIGS["cfg3"]
    x = inputs.points(cfg); y = inputs.rhs(cfg)
    g = hb.HODLR(torch.from_numpy(x).cuda(), cfg.kernel, cfg.theta, cfg.sigma2, cfg.leaf, cfg.eps)
    xg, _ = g.factor_solve(torch.from_numpy(y).cuda())
    xg = xg.cpu().numpy()
    ld_g = g.logdet()
    o = OracleHODLR(x, cfg.kernel, cfg.theta, cfg.sigma2, cfg.leaf, cfg.eps).factor()
    xo = o.solve(y)
    rel = np.linalg.norm(xg - xo) / np.linalg.norm(xo)
    print(f"[full cfg3 eps=1e-10 fused] logdet rel {abs(ld_g - o.logdet()) / abs(o.logdet()):.2e} solve rel {rel:.2e}")
    assert abs(ld_g - o.logdet()) <= LD_TOL * abs(o.logdet())
    assert rel <= X_TOL
    rows = np.random.default_rng(123).choice(cfg.n, 64, replace=False)
    r_g = residual_rows_torch(x, y, xg, rows, cfg.kernel, cfg.a, cfg.ell, cfg.sigma2)
    r_o = residual_rows_torch(x, y, xo, rows, cfg.kernel, cfg.a, cfg.ell, cfg.sigma2)
    assert np.linalg.norm(r_g) <= 2 * np.linalg.norm(r_o)


def residual_rows_torch(x, y, sol, rows, kernel, a, ell, s2):
    """(C sol - y)[rows] with C assembled entry by entry (plain torch fp64 on the GPU: test-side arithmetic, the
    same Table I formula as the oracle's O3)."""
    xs = torch.from_numpy(x).cuda(); s = torch.from_numpy(sol).cuda()
    out = []
    for i in rows:
        d = xs[int(i)] - xs
        assert kernel == 0
        ci = a * a * torch.exp(-(d * d) / (2 * ell * ell))
        ci[int(i)] += s2
        out.append(float(ci @ s) - y[int(i)])
    return np.array(out)


def test_full_size_cfg5_vs_oracle_golden(hb):
    """BASELINE.json config 5 at full size (n = 2^23, 5% clustered duplicates) against the oracle at the parity
    eps = 1e-12, via tests/golden/cfg5_eps1e-12.npz (written by tools/make_golden.py, which calls only oracle/: the
    oracle needs ~17 min and ~45 GB here).  (a) With the oracle's per-block ranks (hodlr_opts.forced_ranks): log det
    <= 1e-9 and the 4096 sampled solution entries <= 1e-9 relative (arithmetic parity).  (b) With the GPU's own ACA
    ranks (a handful of the 65535 blocks differ, R17): the same gates, and the exact residual on 128
    sampled rows within 2x the oracle's own residual on the same rows."""
    import hashlib
    import os
    gold = np.load(os.path.join(os.path.dirname(__file__), "golden", "cfg5_eps1e-12.npz"))
    cfg = inputs.CONFIGS["cfg5"]
    x = inputs.points(cfg); y = inputs.rhs(cfg)
    assert hashlib.sha256(x.tobytes()).hexdigest() == str(gold["x_sha256"])
    assert hashlib.sha256(y.tobytes()).hexdigest() == str(gold["y_sha256"])
    idx = gold["idx"]; xo = gold["x_at_idx"]; ld_o = float(gold["logdet"])
    xd = torch.from_numpy(x).cuda(); yd = torch.from_numpy(y).cuda()
    res = {}
    for mode in ("forced", "free"):
        g = hb.HODLR(xd, cfg.kernel, cfg.theta, cfg.sigma2, cfg.leaf, 1e-12, 64,
                     forced_ranks=gold["ranks"] if mode == "forced" else None)
        xg, _ = g.factor_solve(yd)
        xg = xg.cpu().numpy()
        ld_g = g.logdet()
        r_g = g.tree()[2]
        if mode == "forced":
            np.testing.assert_array_equal(r_g, gold["ranks"])
        g.close()
        rel = np.linalg.norm(xg[idx] - xo) / np.linalg.norm(xo)
        res[mode] = (abs(ld_g - ld_o) / abs(ld_o), rel, xg)
        print(f"[cfg5 full {mode} ranks] logdet rel {res[mode][0]:.2e} sampled solve rel {rel:.2e} rank mismatches {int(np.sum(r_g != gold['ranks']))}")
        assert abs(ld_g - ld_o) <= LD_TOL * abs(ld_o)
    assert res["forced"][1] <= X_TOL
    assert res["free"][1] <= X_TOL
    r_g = residual_rows_torch(x, y, res["free"][2], gold["res_idx"], cfg.kernel, cfg.a, cfg.ell, cfg.sigma2)
    r_o = gold["res_oracle"]
    print(f"[cfg5 full] residual rows: gpu {np.linalg.norm(r_g):.3e} oracle {np.linalg.norm(r_o):.3e}")
    assert np.linalg.norm(r_g) <= 2 * np.linalg.norm(r_o)


def test_full_size_cfg5_shuffled_input_bitwise(hb):
    """Config 5 at full size (n = 2^23, eps = 1e-10): a shuffled copy of the input gives a bitwise-identical log
    det and the same solution permuted (the stable sort makes the factorization independent of the input order,
    ties included)."""
    cfg = inputs.CONFIGS["cfg5"]
    x = inputs.points(cfg); y = inputs.rhs(cfg)
    xd = torch.from_numpy(x).cuda(); yd = torch.from_numpy(y).cuda()
    g = hb.HODLR(xd, cfg.kernel, cfg.theta, cfg.sigma2, cfg.leaf, cfg.eps)
    s1, _ = g.factor_solve(yd); ld1 = g.logdet(); s1 = s1.cpu().numpy(); g.close()
    perm = np.random.default_rng(321).permutation(cfg.n)
    pd = torch.from_numpy(perm).cuda()
    g2 = hb.HODLR(xd[pd].contiguous(), cfg.kernel, cfg.theta, cfg.sigma2, cfg.leaf, cfg.eps)
    s2, _ = g2.factor_solve(yd[pd].contiguous()); ld2 = g2.logdet(); s2 = s2.cpu().numpy(); g2.close()
    assert ld2 == ld1
    np.testing.assert_array_equal(s2, s1[perm])


def test_full_size_cfg3_parity_eps12(hb):
    """Config 3 at full size (n = 2^20) at the parity epsilon 1e-12 (north_star): log det and solve <= 1e-9 relative to
    the oracle (measured 2e-14 and 1.8e-10, every per-block ACA rank equal to the oracle's; the twin floor is
    2.4e-10, R15), and the GPU solution's exact residual on sampled rows (computed one by one on the CPU)
    within 2x the oracle's on the same rows."""
    cfg = inputs.CONFIGS["cfg3"]
    x = inputs.points(cfg); y = inputs.rhs(cfg)
    o, g, ro, rg = run_both(hb, x, y, cfg.kernel, cfg.theta, cfg.sigma2, cfg.leaf, 1e-12)
    ld_o, x_o, _ = ro
    ld_g, x_g, _ = rg
    assert abs(ld_g - ld_o) <= LD_TOL * abs(ld_o)
    rel = np.linalg.norm(x_g - x_o) / np.linalg.norm(x_o)
    print(f"[full cfg3 eps=1e-12] logdet rel {abs(ld_g - ld_o) / abs(ld_o):.2e} solve rel {rel:.2e}")
    assert rel <= X_TOL
    rows = np.random.default_rng(7).choice(cfg.n, 48, replace=False)
    rg_, ro_ = [], []
    for i in rows:
        ci = np.exp(-(x[i] - x) ** 2 / (2 * cfg.ell ** 2)) * cfg.a ** 2
        ci[i] += cfg.sigma2
        rg_.append(ci @ x_g - y[i]); ro_.append(ci @ x_o - y[i])
    assert np.linalg.norm(rg_) <= 2 * np.linalg.norm(ro_) + 1e-12 * np.linalg.norm(y[rows])


def test_cfg5_duplicates_2e18(hb):
    """Config 5 shape (5% clustered duplicates, jitter 1e-6, SE ell = 2 on the config's density) at n = 2^18."""
    cfg = inputs.scaled(inputs.CONFIGS["cfg5"], 1 << 18)
    x = inputs.points(cfg); y = inputs.rhs(cfg)
    o, g, ro, rg = run_both(hb, x, y, cfg.kernel, cfg.theta, cfg.sigma2, cfg.leaf, 1e-12)
    check_parity(o, g, ro, rg)


def test_rank_cap_change_same_shape(hb):
    """the cached ACA plan of a shape must not be reused across rank caps (the factor slot layout
    depends on the cap).  Same n > 2 ACA_FUSED_MAX shape built with cap 48, then 64, then 48 again: every build
    matches the oracle."""
    cfg = inputs.scaled(inputs.CONFIGS["cfg3"], 1 << 15)
    x = inputs.points(cfg); y = inputs.rhs(cfg)
    o = OracleHODLR(x, cfg.kernel, cfg.theta, cfg.sigma2, cfg.leaf, 1e-12).factor()
    ld_o = o.logdet(); x_o = o.solve(y)
    for cap in (48, 64, 48, 20):
        g = hb.HODLR(torch.from_numpy(x).cuda(), cfg.kernel, cfg.theta, cfg.sigma2, cfg.leaf, 1e-12, cap).factor()
        ld_g = g.logdet(); x_g = g.solve(torch.from_numpy(y).cuda()).cpu().numpy()
        g.close()
        assert abs(ld_g - ld_o) <= LD_TOL * abs(ld_o), cap
        assert np.linalg.norm(x_g - x_o) <= X_TOL * np.linalg.norm(x_o), cap


def test_rank_cap_boundary_big_blocks(hb):
    """Lagged stop test of the big-block passes at the rank cap (the dots-only step): with the cap equal to the
    largest oracle rank (held by a big block, sides > ACA_FUSED_MAX) the build succeeds with the oracle's ranks; one
    below it, both the oracle and the GPU return ERANKCAP (the oracle's step 6 after its stop test)."""
    from oracle import OracleError
    cfg = inputs.scaled(inputs.CONFIGS["cfg3"], 1 << 15)
    x = inputs.points(cfg); y = inputs.rhs(cfg)
    o = OracleHODLR(x, cfg.kernel, cfg.theta, cfg.sigma2, cfg.leaf, 1e-12).factor()
    r_o = o.ranks()
    R = int(r_o.max())
    assert int(r_o[:3].max()) == R            # blocks 0..2 (sides 16384, 8192, 8192) run in the passes
    xd = torch.from_numpy(x).cuda()
    g = hb.HODLR(xd, cfg.kernel, cfg.theta, cfg.sigma2, cfg.leaf, 1e-12, R).factor()
    np.testing.assert_array_equal(g.tree()[2][:3], r_o[:3])
    assert abs(g.logdet() - o.logdet()) <= LD_TOL * abs(o.logdet())
    g.close()
    with pytest.raises(OracleError) as eo:
        OracleHODLR(x, cfg.kernel, cfg.theta, cfg.sigma2, cfg.leaf, 1e-12, R - 1)
    assert eo.value.status == "ERANKCAP"
    with pytest.raises(hb.HodlrError) as e:
        hb.HODLR(xd, cfg.kernel, cfg.theta, cfg.sigma2, cfg.leaf, 1e-12, R - 1)
    assert e.value.status == "ERANKCAP"


def test_forced_ranks_hook(hb):
    """hodlr_opts.forced_ranks: the GPU reproduces the oracle's per-block ranks exactly, and with them the solve
    difference is the arithmetic alone (far below the 1e-9 gate)."""
    cfg = inputs.scaled(inputs.CONFIGS["cfg3"], 1 << 16)
    x = inputs.points(cfg); y = inputs.rhs(cfg)
    o = OracleHODLR(x, cfg.kernel, cfg.theta, cfg.sigma2, cfg.leaf, 1e-12).factor()
    r_o = o.ranks()
    g = hb.HODLR(torch.from_numpy(x).cuda(), cfg.kernel, cfg.theta, cfg.sigma2, cfg.leaf, 1e-12, 64,
                 forced_ranks=r_o).factor()
    np.testing.assert_array_equal(g.tree()[2], r_o)
    x_g = g.solve(torch.from_numpy(y).cuda()).cpu().numpy(); x_o = o.solve(y)
    rel = np.linalg.norm(x_g - x_o) / np.linalg.norm(x_o)
    print(f"[forced ranks n=2^16] solve rel {rel:.2e}")
    assert rel <= X_TOL
    assert abs(g.logdet() - o.logdet()) <= LD_TOL * abs(o.logdet())


def test_aca_nograph_identical():
    """HODLR_ACA_NOGRAPH=1 (the profiling switch: host-driven ACA passes instead of the conditional-while graph) runs
    the same kernels: bitwise-identical log det and solution (separate process, the switch is read once)."""
    import os
    import subprocess
    import sys
    code = ("import sys, numpy as np, torch; sys.path.insert(0, '.');"
            "from paper_1403_6015_b200 import inputs; import paper_1403_6015_b200.hodlr as hb;"
            "c = inputs.scaled(inputs.CONFIGS['cfg3'], 1 << 15); x = torch.from_numpy(inputs.points(c)).cuda();"
            "y = torch.from_numpy(inputs.rhs(c)).cuda(); h = hb.HODLR(x, c.kernel, c.theta, c.sigma2, c.leaf, 1e-12);"
            "s, q = h.factor_solve(y); print(repr(h.logdet()), repr(q), float(s.abs().sum()))")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = []
    for ng in ("0", "1"):
        env = dict(os.environ, HODLR_ACA_NOGRAPH=ng)
        outs.append(subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True, text=True,
                                   timeout=300).stdout.strip())
    assert outs[0] and outs[0] == outs[1], outs


@pytest.mark.parametrize("name,n,nrhs", [("cfg1", 2048, 40), ("cfg3", 1 << 15, 33), ("cfg2", 1 << 14, 7)])
def test_batched_multi_rhs(hb, name, n, nrhs):
    """hodlr_solve with many right-hand sides (up to 32 per launch; the leaves take 8 columns per DMMA pass, the tree
    levels run (node, column) pairs) against the oracle's multi-RHS solve, column by column, and against the same
    columns solved one at a time (the single-column leaf path sums in another order: rounding-level agreement)."""
    cfg = inputs.scaled(inputs.CONFIGS[name], n)
    x = inputs.points(cfg, sort=False)
    Y = np.random.default_rng(5).standard_normal((n, nrhs))
    o = OracleHODLR(x, cfg.kernel, cfg.theta, cfg.sigma2, cfg.leaf, 1e-12).factor()
    Xo = o.solve(Y)
    g = hb.HODLR(torch.from_numpy(x).cuda(), cfg.kernel, cfg.theta, cfg.sigma2, cfg.leaf, 1e-12).factor()
    Xg = g.solve(torch.from_numpy(Y).cuda()).cpu().numpy()
    for j in range(nrhs):
        assert np.linalg.norm(Xg[:, j] - Xo[:, j]) <= X_TOL * np.linalg.norm(Xo[:, j]), j
    for j in (0, nrhs // 2, nrhs - 1):
        one = g.solve(torch.from_numpy(np.ascontiguousarray(Y[:, j])).cuda()).cpu().numpy()
        assert np.linalg.norm(one - Xg[:, j]) <= 1e-11 * np.linalg.norm(one), (j, np.linalg.norm(one - Xg[:, j]))
