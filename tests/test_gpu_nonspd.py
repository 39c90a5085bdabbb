"""GPU parity for the kernels that are not positive definite (NEXT-2, R20): multiquadric (sec. 5.2,
Table III) and biharmonic (sec. 5.4, Table VI) on the paper's U[-3, 3]
geometry.  LU leaves (k_leaf_factor_lu), coupling systems of either sign, the signed log det (hodlr_logdet_sign)
against the oracle's (O5' + O8): log |det| <= 1e-9 relative, the sign equal, the solve within max(1e-9, 10 floor)
(floor: the oracle against its Q15 twin, the same compression with QR coupling systems), the ordering and tree
bit-exact."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import MQ, BIHARM, OracleHODLR  # noqa: E402

LD_TOL = 1e-9
X_TOL = 1e-9


@pytest.fixture(scope="module")
def hb():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1403_6015_b200.hodlr as hb
    hb.load()
    return hb


def both(hb, x, y, kernel, theta, s2, leaf, eps=1e-12):
    o = OracleHODLR(x, kernel, theta, s2, leaf, eps).factor()
    t = OracleHODLR(x, kernel, theta, s2, leaf, eps, twin=True).factor()
    la_o, sg_o = o.logdet_sign()
    x_o = o.solve(y)
    floor = float(np.linalg.norm(t.solve(y) - x_o) / np.linalg.norm(x_o))
    xd = torch.from_numpy(x).cuda(); yd = torch.from_numpy(y).cuda()
    g = hb.HODLR(xd, kernel, theta, s2, leaf, eps).factor()
    la_g, sg_g = g.logdet_sign()
    x_g = g.solve(yd).cpu().numpy()
    rel = float(np.linalg.norm(x_g - x_o) / np.linalg.norm(x_o))
    gate = max(X_TOL, 10 * floor)
    print(f"[nonspd k={kernel} n={x.size} s2={s2}] sign {sg_g}/{sg_o} log|det| rel {abs(la_g - la_o) / abs(la_o):.2e} "
          f"solve rel {rel:.2e} (floor {floor:.2e}, gate {gate:.2e})")
    assert sg_g == sg_o
    assert abs(la_g - la_o) <= LD_TOL * abs(la_o)
    assert g.logdet() == la_g
    assert rel <= gate
    xs_g, perm_g = g.order()
    np.testing.assert_array_equal(perm_g.cpu().numpy(), o.perm())
    lo_g, hi_g, r_g = g.tree()
    lo_o, hi_o = o.tree()
    np.testing.assert_array_equal(lo_g, lo_o)
    np.testing.assert_array_equal(hi_g, hi_o)
    r_o = o.ranks()
    if len(r_o):
        assert np.mean(r_g != r_o) <= 0.25 and np.all(np.abs(r_g.astype(int) - r_o.astype(int)) <= 2)
    return o, g, x_o, yd


CASES = [   # (kernel, s2, n, leaf): Table III MQ sigma^2 = 1, Table VI biharmonic sigma^2 = 2
    (MQ, 1.0, 1500, 64),
    (MQ, 1.0, 3000, 64),
    (BIHARM, 2.0, 1500, 64),
    (BIHARM, 2.0, 4097, 128),
    (MQ, 1.0, 1 << 14, 128),
    (BIHARM, 2.0, 3001, 37),
]


@pytest.mark.parametrize("kernel,s2,n,leaf", CASES, ids=[f"{'mq' if c[0] == MQ else 'bh'}-{c[2]}-{c[3]}" for c in CASES])
def test_nonspd_parity(hb, kernel, s2, n, leaf):
    rng = np.random.default_rng(60 + kernel + n)
    x = rng.uniform(-3, 3, n); y = rng.standard_normal(n)
    o, g, x_o, yd = both(hb, x, y, kernel, (1.0, 1.0), s2, leaf)
    with pytest.raises(hb.HodlrError) as e:         # not a covariance: no log-likelihood
        g.gp_loglik(yd)
    assert e.value.status == "EINVAL"
    g.close()


def test_nonspd_both_signs(hb):
    """C = s2 I + MQ on U[-3, 3] has a handful of negative eigenvalues, so det C takes either sign with the shift: the
    GPU's sign equals the oracle's in both cases (cf. tests/test_oracle_pins.py::test_nonspd_sign_both_ways)."""
    rng = np.random.default_rng(0)
    seen = set()
    for n, s2 in ((500, 1.0), (500, 0.5), (1000, 0.5), (1000, 1.0)):
        x = rng.uniform(-3, 3, n); y = rng.standard_normal(n)
        _, g, _, _ = both(hb, x, y, MQ, (1.0, 1.0), s2, 32)
        seen.add(g.logdet_sign()[1])
        g.close()
    assert seen == {1, -1}


def test_nonspd_fused_and_multi_rhs(hb):
    """factor_solve (y fused into the LU-leaf factorization) and a 5-column solve equal the one-column solves."""
    rng = np.random.default_rng(9)
    n = 5000
    x = rng.uniform(-3, 3, n); Y = rng.standard_normal((5, n))
    xd = torch.from_numpy(x).cuda(); Yd = torch.from_numpy(Y).cuda()
    g = hb.HODLR(xd, MQ, (1.0, 1.0), 1.0, 64, 1e-12).factor()
    singles = np.stack([g.solve(Yd[j]).cpu().numpy() for j in range(5)])
    multi = g.solve(Yd.t().contiguous()).cpu().numpy().T          # (n, 5): one launch, the RB = 1 leaf phases
    np.testing.assert_allclose(multi, singles, rtol=0, atol=1e-12 * np.abs(singles).max())
    la, sg = g.logdet_sign()
    g.close()
    h = hb.HODLR(xd, MQ, (1.0, 1.0), 1.0, 64, 1e-12)
    s, quad = h.factor_solve(Yd[0])
    assert h.logdet_sign()[1] == sg and abs(h.logdet() - la) <= 1e-13 * abs(la)
    np.testing.assert_allclose(s.cpu().numpy(), singles[0], rtol=0, atol=1e-11 * np.abs(singles[0]).max())
    assert abs(quad - float(Y[0] @ singles[0])) <= 1e-9 * abs(quad)
    h.close()


def test_nonspd_refusals(hb):
    """Not a covariance: no predictive variance, no sweep; one GPU, unbatched (hodlr.h)."""
    x = torch.linspace(-3, 3, 600, dtype=torch.float64, device="cuda")
    y = torch.ones(600, dtype=torch.float64, device="cuda")
    g = hb.HODLR(x, MQ, (1.0, 1.0), 1.0, 32, 1e-10).factor()
    with pytest.raises(hb.HodlrError):
        g.predict(y, x[:4].clone(), variance=True)
    mean, _ = g.predict(y, x[:4].clone(), variance=False)      # k(xt, x) C^{-1} y (RBF interpolant of the weights)
    xs = x.cpu().numpy(); w = g.solve(y).cpu().numpy()
    ref = np.sqrt(1 + (xs[:4, None] - xs[None, :]) ** 2) @ w
    np.testing.assert_allclose(mean.cpu().numpy(), ref, rtol=1e-9, atol=1e-9 * np.abs(w).sum())
    g.close()
    with pytest.raises(hb.HodlrError):
        hb.HODLRBatch(x, BIHARM, [(1.0, 1.0), (1.0, 1.0)], [2.0, 2.0], 32, 1e-10)


def test_logdet_sign_spd_is_plus_one(hb):
    """hodlr_logdet_sign on an SPD kernel: sign +1 and log |det| = hodlr_logdet (the same factorization)."""
    rng = np.random.default_rng(3)
    x = torch.from_numpy(rng.uniform(0, 10, 4096)).cuda()
    g = hb.HODLR(x, 0, (1.0, 0.5), 1e-2, 64, 1e-10).factor()
    la, sg = g.logdet_sign()
    assert sg == 1 and la == g.logdet()
    g.close()
