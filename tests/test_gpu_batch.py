"""Batched factorizations (hodlr_build_batch, NEXT-4): B = 2^t settings on the same points held as one
block-diagonal handle.  Every problem must reproduce its own single-setting handle (same tree below the problem
root, same blocks, same kernels: the ranks are equal and the results agree to summation order) and the oracle;
the config-4 sweep built on it must equal the per-setting values.  Through the C-ABI (ctypes binding)."""
import math

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


def settings(B, seed=44):
    cfg = inputs.CONFIGS["cfg4"]
    ell, s2 = inputs.sweep_settings(cfg, count=B, seed=seed)
    return cfg, np.stack([np.full(B, cfg.a), ell], axis=1), s2


def subtree_ranks(r_batch, t, s, kappa_s):
    """Ranks of problem s's internal nodes (heap order of its own tree) inside the batched tree."""
    out = []
    for dl in range(kappa_s):
        d = t + dl
        base = (1 << d) - 1 + s * (1 << dl)
        out.extend(r_batch[base:base + (1 << dl)])
    return np.array(out, dtype=np.int32)


@pytest.mark.parametrize("B,n", [(2, 4096), (4, 1 << 13), (8, 3000), (16, 2048)])
def test_batch_matches_single(hb, B, n):
    cfg, th, s2 = settings(B)
    c = inputs.scaled(cfg, n)
    x = inputs.points(c); y = inputs.rhs(c)
    xd = torch.from_numpy(x).cuda(); yd = torch.from_numpy(y).cuda()
    yb = yd.repeat(B)
    gb = hb.HODLRBatch(xd, c.kernel, th, s2, c.leaf, 1e-12)
    xb, qtot = gb.factor_solve(yb)
    ld, q = gb.results()
    xb = xb.cpu().numpy().reshape(B, n)
    _, _, rb = gb.tree()
    t = B.bit_length() - 1
    assert np.all(rb[:(1 << t) - 1] == 0)                     # the problem-coupling blocks are zero
    assert abs(gb.logdet() - ld.sum()) <= 1e-12 * np.abs(ld).sum()
    assert abs(qtot - q.sum()) <= 1e-12 * np.abs(q).sum()
    for s in range(B):
        g = hb.HODLR(xd, c.kernel, th[s], s2[s], c.leaf, 1e-12)
        x1, q1 = g.factor_solve(yd)
        x1 = x1.cpu().numpy(); ld1 = g.logdet()
        lo, hi, r1 = g.tree()
        k1 = g.info()["kappa"]
        np.testing.assert_array_equal(subtree_ranks(rb, t, s, k1), r1)
        assert abs(ld[s] - ld1) <= 1e-13 * abs(ld1), (s, ld[s], ld1)
        assert abs(q[s] - q1) <= 1e-12 * abs(q1), (s, q[s], q1)
        assert np.linalg.norm(xb[s] - x1) <= 1e-12 * np.linalg.norm(x1), s
        g.close()
    gb.close()


def test_batch_vs_oracle(hb):
    """Every problem of a 4-setting batch (including the sweep's stiffest corner: ell = 2, sigma2 = 1e-4) against
    the oracle at the parity gates."""
    cfg = inputs.CONFIGS["cfg4"]
    c = inputs.scaled(cfg, 1 << 13)
    x = inputs.points(c); y = inputs.rhs(c)
    th = np.array([[cfg.a, 0.05], [cfg.a, 0.3], [cfg.a, 1.0], [cfg.a, 2.0]])
    s2 = np.array([0.1, 1e-2, 1e-3, 1e-4])
    gb = hb.HODLRBatch(torch.from_numpy(x).cuda(), c.kernel, th, s2, c.leaf, 1e-12)
    xb, _ = gb.factor_solve(torch.from_numpy(y).cuda().repeat(4))
    ld, q = gb.results()
    xb = xb.cpu().numpy().reshape(4, -1)
    for s in range(4):
        o = OracleHODLR(x, c.kernel, th[s], s2[s], c.leaf, 1e-12).factor()
        ld_o = o.logdet(); x_o = o.solve(y)
        rel = np.linalg.norm(xb[s] - x_o) / np.linalg.norm(x_o)
        print(f"[batch vs oracle] setting {s}: logdet rel {abs(ld[s] - ld_o) / abs(ld_o):.1e} solve rel {rel:.1e}")
        assert abs(ld[s] - ld_o) <= 1e-9 * abs(ld_o)
        assert rel <= 1e-8 if s == 3 else rel <= 1e-9            # the corner's FP64 floor (R15)
        assert abs(q[s] - float(y @ x_o)) <= 1e-8 * abs(float(y @ x_o))


def test_batch_unfused_and_apply(hb):
    """The batched handle through the plain factor / solve / apply path: each problem equals its own handle."""
    cfg, th, s2 = settings(4, seed=7)
    c = inputs.scaled(cfg, 4096)
    x = inputs.points(c)
    rng = np.random.default_rng(3)
    Y = rng.standard_normal(4 * c.n)
    gb = hb.HODLRBatch(torch.from_numpy(x).cuda(), c.kernel, th, s2, c.leaf, 1e-12).factor()
    Yd = torch.from_numpy(Y).cuda()
    Xs = gb.solve(Yd).cpu().numpy().reshape(4, -1)
    AY = gb.apply(Yd).cpu().numpy().reshape(4, -1)
    ld = gb.results(quad=False)
    for s in range(4):
        g = hb.HODLR(torch.from_numpy(x).cuda(), c.kernel, th[s], s2[s], c.leaf, 1e-12).factor()
        ys = torch.from_numpy(Y[s * c.n:(s + 1) * c.n]).cuda()
        x1 = g.solve(ys).cpu().numpy()
        a1 = g.apply(ys).cpu().numpy()
        assert np.linalg.norm(Xs[s] - x1) <= 1e-12 * np.linalg.norm(x1)
        assert np.linalg.norm(AY[s] - a1) <= 1e-14 * np.linalg.norm(a1)
        assert abs(ld[s] - g.logdet()) <= 1e-13 * abs(g.logdet())


def test_batch_errors(hb):
    cfg, th, s2 = settings(4)
    xd = torch.linspace(0, 1, 1000, dtype=torch.float64, device="cuda")
    with pytest.raises(hb.HodlrError) as e:
        hb.HODLRBatch(xd, cfg.kernel, th[:3], s2[:3], 64, 1e-12)            # B = 3: not a power of two
    assert e.value.status == "EINVAL"
    with pytest.raises(hb.HodlrError) as e:
        hb.HODLRBatch(xd[:50], cfg.kernel, th, s2, 64, 1e-12)              # n < leaf
    assert e.value.status == "EINVAL"
    bad = s2.copy(); bad[2] = -1.0
    with pytest.raises(hb.HodlrError) as e:
        hb.HODLRBatch(xd, cfg.kernel, th, bad, 64, 1e-12)
    assert e.value.status == "EINVAL" and "setting 2" in str(e.value)
    gb = hb.HODLRBatch(xd, cfg.kernel, th, s2, 64, 1e-12)
    with pytest.raises(hb.HodlrError) as e:
        gb.results()
    assert e.value.status == "ESTATE"
    gb.factor()
    with pytest.raises(hb.HodlrError) as e:
        gb.results()                                                         # no right-hand side fused
    assert e.value.status == "ESTATE"
    with pytest.raises(hb.HodlrError) as e:
        gb.predict(torch.zeros(4 * 1000, dtype=torch.float64, device="cuda"), xd[:4])
    assert e.value.status == "EINVAL"


def test_sweep_batched_with_failing_setting(hb):
    """gp_loglik_sweep over 8 settings where one is not positive definite (sigma2 = 0 on exact duplicates): the
    batch fails, is redone setting by setting, and only that setting reports -inf."""
    x = np.repeat(np.linspace(0.0, 10.0, 1024), 2)
    y = np.random.default_rng(0).standard_normal(x.size)
    th = np.array([[1.0, 0.3]] * 8)
    s2 = np.full(8, 1e-2); s2[5] = 0.0
    xd = torch.from_numpy(x).cuda(); yd = torch.from_numpy(y).cuda()
    with pytest.raises(hb.HodlrError) as e:
        hb.gp_loglik_sweep(xd, yd, hb.HODLR_MATERN52, th, s2, 64, 1e-10)
    vals = e.value.values
    assert e.value.status == "ENOTPD" and "setting 5" in str(e.value)
    assert np.isneginf(vals[5]) and np.all(np.isfinite(np.delete(vals, 5)))
    one = hb.HODLR(xd, hb.HODLR_MATERN52, th[0], 1e-2, 64, 1e-10).factor().gp_loglik(yd)
    assert abs(vals[0] - one) <= 1e-12 * abs(one)


def test_sweep_full_cfg4_vs_single(hb):
    """Config 4 at full size (n = 131072, 64 settings in one batched handle): every value equals the
    single-setting fused path to 1e-12 (summation order only) -- 8 settings sampled, including the stiffest."""
    cfg = inputs.CONFIGS["cfg4"]
    ell, s2 = inputs.sweep_settings(cfg)
    x = inputs.points(cfg); y = inputs.rhs(cfg)
    th = np.stack([np.full(64, cfg.a), ell], axis=1)
    xd = torch.from_numpy(x).cuda(); yd = torch.from_numpy(y).cuda()
    vals = hb.gp_loglik_sweep(xd, yd, cfg.kernel, th, s2, cfg.leaf, cfg.eps)
    worst = int(np.argmax(ell / np.sqrt(s2)))
    for k in sorted({0, 13, 31, 40, 63, worst, int(np.argmin(s2)), int(np.argmax(ell))}):
        g = hb.HODLR(xd, cfg.kernel, th[k], s2[k], cfg.leaf, cfg.eps)
        _, quad = g.factor_solve(yd, solve=False)
        one = -0.5 * quad - 0.5 * g.logdet() - 0.5 * cfg.n * math.log(2 * math.pi)
        g.close()
        assert abs(vals[k] - one) <= 1e-12 * abs(one), (k, vals[k], one)
