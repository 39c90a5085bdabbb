"""Pins for the CPU oracle (-m "not gpu").

The oracle (oracle/hodlr_oracle.c) is checked against things other than
itself: closed forms, brute-force dense linear algebra (numpy/scipy, an
independent code path), exact invariants, and special cases that reduce to a
textbook identity.  Each test names the plausible mistake it would catch.
"""
import math
import os

import numpy as np
import pytest
import scipy.special as sps

from oracle import (SE, MATERN32, MATERN52, EXP, IMQ, RQ, OracleHODLR, OracleError, aca_dense, dense_check,
                    kernel_value)

GOLD = {}
with open(os.path.join(os.path.dirname(__file__), "golden", "closed_forms.txt")) as f:
    for line in f:
        line = line.split("#")[0].strip()
        if line:
            k, v = line.split()
            GOLD[k] = float(v)


def dense_C(x, kernel, theta, s2):
    """Independent numpy assembly of C = s2 I + K (Table I formulas)."""
    a, ell = theta[0], theta[1]
    d = np.abs(x[:, None] - x[None, :])
    if kernel == SE:
        K = a * a * np.exp(-d * d / (2 * ell * ell))
    elif kernel == EXP:      # Table I Ornstein-Uhlenbeck = Matern-1/2 (Bessel form with nu = 1/2)
        z = d / ell
        with np.errstate(invalid="ignore"):
            K = a * a * (2 ** 0.5 / sps.gamma(0.5)) * z ** 0.5 * sps.kv(0.5, z)
        K[d == 0] = a * a
    elif kernel in (IMQ, RQ):  # rational quadratic (IMQ: alpha = 1/2) via exp(-alpha log1p(.))
        alpha = 0.5 if kernel == IMQ else theta[2]
        K = a * a * np.exp(-alpha * np.log1p((d / ell) ** 2))
    else:   # Table I Matern through the Bessel form -- a different formula from the oracle's closed form
        nu = 1.5 if kernel == MATERN32 else 2.5
        z = np.sqrt(2 * nu) * d / ell
        with np.errstate(invalid="ignore"):
            K = a * a * (2 ** (1 - nu) / sps.gamma(nu)) * z ** nu * sps.kv(nu, z)
        K[d == 0] = a * a
    return K + s2 * np.eye(len(x))


# ---------------------------------------------------------------- O1/O2
@pytest.mark.parametrize("n,p,kappa", [(16, 20, 0), (10000, 20, 8), (2048, 64, 5), (1 << 20, 128, 13),
                                       (1000000, 128, 12), (1, 1, 0), (2, 1, 1), (127, 64, 0), (128, 64, 1)])
def test_kappa_formula(n, p, kappa):
    """Fig. 6 line 1 kappa = floor(log2(n/p_max))."""
    x = np.linspace(0, 1, n)
    h = OracleHODLR(x, SE, (1.0, 1.0), 1.0, p, 1e-6)
    assert h.kappa == kappa
    lo, hi = h.tree()
    assert len(lo) == 2 ** (kappa + 1) - 1


@pytest.mark.parametrize("n,p", [(1000, 20), (999, 64), (2048, 64), (777, 7), (64, 64)])
def test_tree_invariants(n, p):
    """Count-median tree: levels tile [0,n), siblings differ by <= 1 (left = ceil), leaves in [p, 2p)."""
    x = np.random.default_rng(0).uniform(0, 1, n)
    h = OracleHODLR(x, SE, (1.0, 0.1), 1.0, p, 1e-6)
    lo, hi = h.tree()
    kap = h.kappa
    for d in range(kap + 1):
        ids = np.arange(2 ** d - 1, 2 ** (d + 1) - 1)
        assert lo[ids[0]] == 0 and hi[ids[-1]] == n
        assert np.all(lo[ids[1:]] == hi[ids[:-1]])
    for c in range(2 ** kap - 1):
        m1 = hi[2 * c + 1] - lo[2 * c + 1]; m2 = hi[2 * c + 2] - lo[2 * c + 2]
        assert m1 - m2 in (0, 1)
    leaves = hi[2 ** kap - 1:] - lo[2 ** kap - 1:]
    if n >= p:
        assert leaves.min() >= p and leaves.max() < 2 * p


def test_sort_is_stable_argsort():
    """O1: perm = stable ascending argsort (ties by original index), -0.0 canonicalised."""
    rng = np.random.default_rng(5)
    x = rng.integers(0, 50, 3000).astype(np.float64) * 0.25 - 3.0
    x[::97] = -0.0
    x[1::97] = 0.0
    h = OracleHODLR(x, SE, (1.0, 1.0), 1.0, 20, 1e-6)
    xc = np.where(x == 0.0, 0.0, x)
    np.testing.assert_array_equal(h.perm(), np.argsort(xc, kind="stable"))
    np.testing.assert_array_equal(h.sorted_x(), np.sort(xc))
    assert not np.any(np.signbit(h.sorted_x()[h.sorted_x() == 0.0]))


# ---------------------------------------------------------------- O3
def test_kernel_closed_forms_golden():
    """Table I values at r = ell (golden file, hand-derived)."""
    assert kernel_value(SE, (1.0, 1.0), 1.0) == pytest.approx(GOLD["se_at_r_eq_ell"], rel=1e-15)
    assert kernel_value(MATERN32, (1.0, 1.0), 1.0) == pytest.approx(GOLD["matern32_at_r_eq_ell"], rel=1e-15)
    assert kernel_value(MATERN52, (1.0, 1.0), 1.0) == pytest.approx(GOLD["matern52_at_r_eq_ell"], rel=1e-15)
    for k in (SE, MATERN32, MATERN52):
        assert kernel_value(k, (2.0, 0.3), 0.0) == 4.0          # a^2 at r = 0 (removable singularity)


@pytest.mark.parametrize("kernel,nu", [(MATERN32, 1.5), (MATERN52, 2.5)])
def test_matern_matches_bessel_form(kernel, nu):
    """Table I Matern sigma^2 (sqrt(2nu) r)^nu K_nu(sqrt(2nu) r) / (Gamma(nu) 2^(nu-1)) via scipy.special.kv."""
    a, ell = 1.3, 0.7
    for r in np.geomspace(1e-3, 30, 200):
        z = math.sqrt(2 * nu) * r / ell
        ref = a * a * z ** nu * sps.kv(nu, z) / (sps.gamma(nu) * 2 ** (nu - 1))
        assert kernel_value(kernel, (a, ell), r) == pytest.approx(ref, rel=2e-13, abs=1e-300)


def test_kernel_symmetry_and_se_scaling():
    """k(d) = k(-d) exactly; SE with ell=1/sqrt(2) is Table II's exp(-r^2)."""
    for k in (SE, MATERN32, MATERN52):
        for d in np.linspace(-5, 5, 101):
            assert kernel_value(k, (1.0, 0.9), d) == kernel_value(k, (1.0, 0.9), -d)
    for d in np.linspace(0, 4, 41):
        assert kernel_value(SE, (1.0, 1 / math.sqrt(2)), d) == pytest.approx(math.exp(-d * d), rel=1e-14)


# ---------------------------------------------------------------- O4
def test_aca_rank1_exact():
    """A_ij = x_i y_j with power-of-two entries (exact products): the second residual row is exactly 0,
    so ACA stops at rank 1 with exact reconstruction."""
    rng = np.random.default_rng(1)
    x = 2.0 ** rng.integers(-4, 4, 40); y = 2.0 ** rng.integers(-4, 4, 33)
    A = np.outer(x, y)
    U, V, r = aca_dense(A, 1e-12)
    assert r == 1
    np.testing.assert_array_equal(U @ V.T, A)


def test_aca_rank1_generic():
    """Generic rank-1 source: the kept stopping term is a rounding-level second term (R4),
    so rank <= 2 and the reconstruction is exact to rounding."""
    rng = np.random.default_rng(1)
    x = rng.uniform(0.5, 2, 40); y = rng.uniform(0.5, 2, 33)
    A = np.outer(x, y)
    U, V, r = aca_dense(A, 1e-12)
    assert r <= 2
    np.testing.assert_allclose(U @ V.T, A, rtol=1e-15, atol=1e-15)


def test_aca_zero_block():
    U, V, r = aca_dense(np.zeros((20, 30)), 1e-12)
    assert r == 0


def test_aca_full_rank_stops_at_min():
    """Generic dense 6x7 block: ACA reaches min(m1,m2) = 6 and reproduces the block (partial-pivoted LU)."""
    A = np.random.default_rng(2).standard_normal((6, 7))
    U, V, r = aca_dense(A, 1e-12)
    assert r == 6
    np.testing.assert_allclose(U @ V.T, A, atol=1e-13)


def test_aca_identity_blind_spot():
    """Identity: the pivot column is zero on every unused row, so step 7 stops at rank 1 -- the known
    sampling blind spot of partial pivoting the paper warns about."""
    U, V, r = aca_dense(np.eye(6), 1e-12)
    assert r == 1


def test_aca_rank_cap_error():
    with pytest.raises(OracleError) as e:
        aca_dense(np.random.default_rng(3).standard_normal((8, 8)), 1e-12, cap=3)
    assert e.value.status == "ERANKCAP"


def svd_rank(A, eps):
    s = np.linalg.svd(A, compute_uv=False)
    tail = np.sqrt(np.cumsum((s ** 2)[::-1]))[::-1]   # tail[k] = ||s[k:]||
    fro = np.linalg.norm(s)
    for k in range(len(s) + 1):
        if k == len(s) or tail[k] <= eps * fro:
            return k


@pytest.mark.parametrize("ell,eps", [(0.1, 1e-12), (1.0, 1e-10), (0.05, 1e-8)])
def test_aca_se_block_vs_svd(ell, eps):
    """SE off-diagonal block: rank <= SVD eps-rank + 5 and ||A - UV^T||_F <= 10 eps ||A||_F."""
    rng = np.random.default_rng(3)
    x = np.sort(rng.uniform(0, 1, 1024))
    x1, x2 = x[:512], x[512:]
    A = np.exp(-(x1[:, None] - x2[None, :]) ** 2 / (2 * ell * ell))
    U, V, r = aca_dense(A, eps)
    err = np.linalg.norm(A - U @ V.T) / np.linalg.norm(A)
    assert err <= 10 * eps
    assert r <= svd_rank(A, eps) + 5


@pytest.mark.parametrize("kernel,maxr", [(MATERN32, 3), (MATERN52, 4)])
def test_aca_matern_semiseparable(kernel, maxr):
    """1-D Matern-3/2 (5/2) blocks of sorted points have exact rank 2 (3): ACA stops by rank 3 (4)."""
    rng = np.random.default_rng(4)
    x = np.sort(rng.uniform(0, 10, 800))
    x1, x2 = x[:400], x[400:]
    A = np.array([[kernel_value(kernel, (1.0, 0.5), a - b) for b in x2] for a in x1])
    U, V, r = aca_dense(A, 1e-12)
    assert r <= maxr
    assert np.linalg.norm(A - U @ V.T) <= 1e-11 * np.linalg.norm(A)


# ---------------------------------------------------------------- O5-O10: closed forms
@pytest.mark.parametrize("twin", [False, True], ids=["oracle", "twin"])
def test_two_by_two(twin):
    """One-level example eq-two-level-1: C = [[2,.5],[.5,2]], leaf 1."""
    d = math.sqrt(2 * math.log(2.0))      # SE, a = ell = 1: exp(-d^2/2) = 1/2
    h = OracleHODLR(np.array([0.0, d]), SE, (1.0, 1.0), 1.0, 1, 1e-12, twin=twin).factor()
    assert h.kappa == 1
    assert h.logdet() == pytest.approx(GOLD["twobytwo_logdet"], rel=1e-15)
    x = h.solve(np.array([1.0, -1.0]))
    np.testing.assert_allclose(x, [GOLD["twobytwo_x0"], -GOLD["twobytwo_x0"]], rtol=1e-15)


def test_zero_kernel_closed_form():
    """K = 0 (a = 0): log det = n log s2, x = y / s2, loglik closed form."""
    rng = np.random.default_rng(1)
    n, s2 = 2048, 1e-2
    x = np.sort(rng.uniform(0, 1, n)); y = rng.standard_normal(n)
    h = OracleHODLR(x, SE, (0.0, 0.1), s2, 64, 1e-12).factor()
    assert h.logdet() == pytest.approx(GOLD["zero_kernel_logdet_cfg1"], rel=1e-14)
    np.testing.assert_allclose(h.solve(y), y / s2, rtol=1e-15)
    assert np.all(h.ranks() == 0)
    ll = -0.5 * np.dot(y, y) / s2 - 0.5 * n * math.log(s2) - 0.5 * n * math.log(2 * math.pi)
    assert h.gp_loglik(y) == pytest.approx(ll, rel=1e-13)
    assert h.gp_loglik(np.zeros(n)) == pytest.approx(-0.5 * n * math.log(s2) - 0.5 * n * math.log(2 * math.pi), rel=1e-14)


def test_identity_times_two():
    """C = 2I, n = 100."""
    h = OracleHODLR(np.linspace(0, 1, 100), SE, (0.0, 1.0), 2.0, 8, 1e-12).factor()
    assert h.logdet() == pytest.approx(GOLD["eye2_logdet_n100"], rel=1e-15)


@pytest.mark.parametrize("twin", [False, True], ids=["oracle", "twin"])
def test_rank_one_sylvester(twin):
    """SE with ell = 1e20: K = a^2 11^T exactly.  Sylvester / Sherman-Morrison closed forms."""
    rng = np.random.default_rng(7)
    n, s2 = 1024, 1e-2
    x = rng.uniform(0, 1, n); y = rng.standard_normal(n)
    h = OracleHODLR(x, SE, (1.0, 1e20), s2, 64, 1e-12, twin=twin).factor()
    assert h.logdet() == pytest.approx(GOLD["rank1_logdet_n1024"], rel=1e-13)
    xs = (y - y.sum() / (s2 + n) * np.ones(n)) / s2
    np.testing.assert_allclose(h.solve(y), xs, rtol=1e-10, atol=1e-10 * np.abs(xs).max())
    assert np.all(h.ranks() == 1)


def test_far_separated_clusters_additive():
    """Two clusters 100 apart with SE ell = 0.05: the top block is exactly 0 (rank 0), log det adds."""
    rng = np.random.default_rng(8)
    xa = np.sort(rng.uniform(0, 1, 256)); xb = np.sort(rng.uniform(100, 101, 256))
    x = np.concatenate([xa, xb]); th = (1.0, 0.05); s2 = 1e-2
    h = OracleHODLR(x, SE, th, s2, 32, 1e-12).factor()
    assert h.ranks()[0] == 0
    la = np.linalg.slogdet(dense_C(xa, SE, th, s2))[1]; lb = np.linalg.slogdet(dense_C(xb, SE, th, s2))[1]
    assert h.logdet() == pytest.approx(la + lb, rel=1e-13)


# ---------------------------------------------------------------- dense brute force
CASES = [
    ("cfg1", 2048, 0.0, 1.0, SE, (1.0, 0.1), 1e-2, 64),
    ("cfg3-density", 4096, 0.0, 100.0 * 4096 / 2 ** 20 * 32, SE, (1.0, 1.0), 1e-2, 128),
    ("cfg2-density", 2048, 0.0, 10.0 * 2048 / 65536 * 16, MATERN32, (1.0, 0.5), 1e-3, 64),
    ("cfg4-corner", 2048, 0.0, 10.0 * 2048 / 131072 * 32, MATERN52, (1.0, 2.0), 1e-4, 64),
    ("ragged", 1999, -3.0, 3.0, SE, (1.0, 1 / math.sqrt(2)), 1.0, 50),
    ("m52-ragged", 1531, 0.0, 4.0, MATERN52, (0.8, 0.3), 1e-2, 37),
]


CASES.append(("exact-duplicates", 3000, 0.0, 12.0, SE, (1.3, 0.7), 1e-2, 64))
CASES += [("exp-ou", 2048, 0.0, 8.0, EXP, (1.1, 0.5), 1e-2, 64),            # NEXT-2 kernels (Tables I, IV, V)
          ("imq", 1500, -3.0, 3.0, IMQ, (1.0, 0.3), 1e-1, 40),
          ("rq-1.5", 1800, 0.0, 5.0, RQ, (0.9, 0.4, 1.5), 1e-2, 48)]


@pytest.mark.parametrize("twin", [False, True], ids=["oracle", "twin"])
@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_hodlr_vs_dense(case, twin):
    """log det <= 1e-12 rel and solve <= 1e-9 rel against numpy dense (independent LAPACK path), for the oracle and
    for its Q15 twin (leaf LU + coupling-system QR): a wrong reflection sign, a missed pivot swap or a dropped
    Householder update in the twin fails here."""
    _, n, lo, hi, k, th, s2, p = case
    rng = np.random.default_rng(11)
    x = rng.uniform(lo, hi, n); y = rng.standard_normal(n)
    if case[0] == "exact-duplicates":     # ~2.5 points per distinct value, plus a block of zeros (R2)
        x = np.round(x, 2); x[::97] = 0.0
    h = OracleHODLR(x, k, th, s2, p, 1e-12, twin=twin).factor()
    C = dense_C(x, k, th, s2)
    sd, ld = np.linalg.slogdet(C)
    assert sd > 0
    assert abs(h.logdet() - ld) <= 1e-12 * abs(ld) + 1e-9
    xd = np.linalg.solve(C, y)
    xh = h.solve(y)
    assert np.linalg.norm(xh - xd) <= 1e-9 * np.linalg.norm(xd)
    # O11 dense checker (own loops) agrees with numpy too
    ld2, x2 = dense_check(x, k, th, s2, y)
    assert abs(ld2 - ld) <= 1e-12 * abs(ld)
    assert np.linalg.norm(x2 - xd) <= 1e-9 * np.linalg.norm(xd)
    ll = -0.5 * y @ xd - 0.5 * ld - 0.5 * n * math.log(2 * math.pi)
    assert h.gp_loglik(y) == pytest.approx(ll, rel=1e-10)


@pytest.mark.parametrize("twin", [False, True], ids=["oracle", "twin"])
@pytest.mark.parametrize("n,p,k", [(256, 16, SE), (300, 7, MATERN32), (512, 32, MATERN52)])
def test_factorization_is_exact_inverse_of_hodlr_matrix(n, p, k, twin):
    """Factor-product identity: solve and log det invert the assembled HODLR matrix H
    to rounding level (not to eps), so any dropped term / wrong sign / swapped P,Q fails here."""
    rng = np.random.default_rng(12)
    x = rng.uniform(0, 3, n)
    h = OracleHODLR(x, k, (1.0, 0.4), 1e-2, p, 1e-6, twin=twin).factor()   # loose eps: H differs from C
    H = np.stack([h.apply(e) for e in np.eye(n)], axis=1)
    assert np.array_equal(H, H.T)
    C = dense_C(x, k, (1.0, 0.4), 1e-2)
    assert np.linalg.norm(H - C) <= 1e-4 * np.linalg.norm(C)
    sd, ld = np.linalg.slogdet(H)
    assert abs(h.logdet() - ld) <= 1e-12 * abs(ld)
    Xi = h.solve(H)
    cond = np.linalg.cond(H)
    assert np.linalg.norm(Xi - np.eye(n)) <= 1e-15 * cond * n


def test_permutation_invariance():
    """Shuffled input: bitwise-identical log det, permuted solution."""
    rng = np.random.default_rng(13)
    n = 1500
    x = rng.uniform(0, 5, n); y = rng.standard_normal(n)
    h1 = OracleHODLR(x, MATERN32, (1.0, 0.5), 1e-2, 40, 1e-12).factor()
    pi = rng.permutation(n)
    h2 = OracleHODLR(x[pi], MATERN32, (1.0, 0.5), 1e-2, 40, 1e-12).factor()
    assert h1.logdet() == h2.logdet()
    np.testing.assert_array_equal(h1.solve(y)[pi], h2.solve(y[pi]))


def test_logdet_parts_sum():
    rng = np.random.default_rng(14)
    x = rng.uniform(0, 1, 1000)
    h = OracleHODLR(x, SE, (1.0, 0.1), 1e-2, 30, 1e-12).factor()
    a, b = h.logdet_parts()
    assert math.fsum(list(a) + list(b)) == pytest.approx(h.logdet(), rel=1e-15)


def test_multi_rhs():
    rng = np.random.default_rng(15)
    x = rng.uniform(0, 1, 700); Y = rng.standard_normal((700, 3))
    h = OracleHODLR(x, SE, (1.0, 0.1), 1e-2, 32, 1e-12).factor()
    X = h.solve(Y)
    for j in range(3):
        np.testing.assert_array_equal(X[:, j], h.solve(Y[:, j]))


# ---------------------------------------------------------------- error behaviour
def test_errors():
    x = np.linspace(0, 1, 100)
    for bad in [dict(n_x=np.array([])), dict(leaf=0), dict(eps=0.0), dict(eps=1.0), dict(s2=-1.0),
                dict(theta=(1.0, 0.0)), dict(theta=(-1.0, 1.0)), dict(kernel=8),
                dict(n_x=np.array([0.0, np.nan])), dict(n_x=np.array([np.inf, 1.0]))]:
        args = dict(n_x=x, kernel=SE, theta=(1.0, 0.1), s2=1e-2, leaf=16, eps=1e-12)
        args.update(bad)
        with pytest.raises(OracleError) as e:
            OracleHODLR(args["n_x"], args["kernel"], args["theta"], args["s2"], args["leaf"], args["eps"])
        assert e.value.status == "EINVAL"
    h = OracleHODLR(x, SE, (1.0, 0.1), 1e-2, 16, 1e-12)
    with pytest.raises(OracleError) as e:
        h.solve(np.ones(100))
    assert e.value.status == "ESTATE"
    # duplicate points with s2 = 0: C is singular -> ENOTPD, log det -inf
    hd = OracleHODLR(np.repeat(np.linspace(0, 1, 50), 2), SE, (1.0, 0.1), 0.0, 16, 1e-12)
    with pytest.raises(OracleError) as e:
        hd.factor()
    assert e.value.status == "ENOTPD"
    with pytest.raises(OracleError):
        hd.logdet()


def test_single_point():
    h = OracleHODLR(np.array([0.3]), MATERN52, (2.0, 1.0), 0.5, 64, 1e-12).factor()
    assert h.logdet() == pytest.approx(math.log(4.5), rel=1e-15)
    assert h.solve(np.array([9.0]))[0] == pytest.approx(2.0, rel=1e-15)


# ---------------------------------------------------------------------------------------------------------------
# NEXT-1: GP prediction (eq_reg1 / eq_reg2)
def _cross(xt, x, kernel, theta):
    """Independent numpy cross-covariance k(xt_j, x_i) (same Table I forms as dense_C)."""
    xx = np.concatenate([np.asarray(xt, float), np.asarray(x, float)])
    Cfull = dense_C(xx, kernel, theta, 0.0)
    return Cfull[:len(xt), len(xt):]


@pytest.mark.parametrize("kernel", [SE, MATERN32, MATERN52])
def test_predict_vs_dense_gp(kernel):
    """Oracle predict (HODLR solve + cross-covariances) against the dense GP posterior (numpy LAPACK solve on an
    independently assembled C).  Catches: a wrong sign in the variance, sigma^2 added to the latent variance, a
    transposed cross-covariance, alpha taken in sorted instead of original order."""
    rng = np.random.default_rng(11 + kernel)
    n, theta, s2 = 300, (1.3, 0.35), 1e-2
    x = rng.uniform(0, 3, n); y = rng.standard_normal(n)
    xt = rng.uniform(-0.2, 3.2, 17)
    o = OracleHODLR(x, kernel, theta, s2, 16, 1e-13).factor()
    mean, var = o.predict(y, xt)
    C = dense_C(x, kernel, theta, s2)
    Ks = _cross(xt, x, kernel, theta)
    mean_d = Ks @ np.linalg.solve(C, y)
    var_d = theta[0] ** 2 - np.einsum("ij,ji->i", Ks, np.linalg.solve(C, Ks.T))
    np.testing.assert_allclose(mean, mean_d, rtol=1e-8, atol=1e-10)
    np.testing.assert_allclose(var, var_d, rtol=1e-7, atol=1e-10)


def test_predict_single_point_closed_form():
    """n = 1: mean = k(t - x1) y / (a^2 + s2), var = a^2 - k(t - x1)^2 / (a^2 + s2) exactly (up to rounding)."""
    a, ell, s2, x1, y1 = 1.7, 0.4, 0.3, 0.25, -1.2
    o = OracleHODLR(np.array([x1]), SE, (a, ell), s2, 8, 1e-12).factor()
    xt = np.array([0.25, 0.1, 1.5])
    mean, var = o.predict(np.array([y1]), xt)
    k = a * a * np.exp(-(xt - x1) ** 2 / (2 * ell * ell))
    np.testing.assert_allclose(mean, k * y1 / (a * a + s2), rtol=1e-14)
    np.testing.assert_allclose(var, a * a - k * k / (a * a + s2), rtol=1e-13, atol=1e-15)


@pytest.mark.parametrize("kernel,theta,expect", [
    (EXP, (1.3, 0.7), 1.3 ** 2 * math.exp(-1.0)),          # d = ell: a^2 e^-1
    (IMQ, (1.3, 0.7), 1.3 ** 2 / math.sqrt(2.0)),          # d = ell: a^2 / sqrt 2
    (RQ, (1.3, 0.7, 1.5), 1.3 ** 2 * 2.0 ** -1.5),         # d = ell: a^2 2^-alpha
])
def test_next2_kernel_closed_forms(kernel, theta, expect):
    """NEXT-2 covariance functions at d = ell and d = 0 (closed forms): a wrong scale (ell vs ell^2, 2 ell^2), a
    missing amplitude or exponent sign fails."""
    assert kernel_value(kernel, theta, theta[1]) == pytest.approx(expect, rel=1e-15)
    assert kernel_value(kernel, theta, -theta[1]) == pytest.approx(expect, rel=1e-15)
    assert kernel_value(kernel, theta, 0.0) == pytest.approx(theta[0] ** 2, rel=1e-15)


def test_rq_alpha_half_is_imq():
    for d in (0.0, 0.1, 1.7, -4.0):
        assert kernel_value(RQ, (1.2, 0.6, 0.5), d) == pytest.approx(kernel_value(IMQ, (1.2, 0.6), d), rel=1e-15)
    with pytest.raises(OracleError):
        OracleHODLR(np.linspace(0, 1, 10), RQ, (1.0, 0.5, -1.0), 1e-2, 4, 1e-10)


# ---------------------------------------------------------------------------------------------------------------
# Q15 oracle twin: leaf LU + coupling-system Householder QR; same compression
def test_twin_shares_compression_and_differs_only_by_rounding():
    """The twin runs the same sort / tree / ACA (identical ranks and tree), so its log det and solve differ from
    the oracle's only by the rounding of two backward-stable dense factorizations.  A twin that silently fell back
    to the oracle's own Cholesky / LU would give a bitwise-equal solve: the difference must be nonzero (at this
    conditioning) and tiny."""
    rng = np.random.default_rng(21)
    n = 4096
    x = rng.uniform(0.0, 10.0 * 4096 / 131072 * 32, n); y = rng.standard_normal(n)
    o = OracleHODLR(x, MATERN52, (1.0, 2.0), 1e-4, 64, 1e-12).factor()
    t = OracleHODLR(x, MATERN52, (1.0, 2.0), 1e-4, 64, 1e-12, twin=True).factor()
    np.testing.assert_array_equal(o.ranks(), t.ranks())
    xo, xt = o.solve(y), t.solve(y)
    d = np.linalg.norm(xo - xt) / np.linalg.norm(xo)
    assert 0.0 < d <= 1e-8
    assert abs(o.logdet() - t.logdet()) <= 1e-12 * abs(o.logdet())
    la_o, nb_o = o.logdet_parts(); la_t, nb_t = t.logdet_parts()
    np.testing.assert_allclose(la_t, la_o, rtol=1e-12)       # leaf LU log|det| = Cholesky 2 sum log L_ii
    np.testing.assert_allclose(nb_t, nb_o, rtol=1e-9, atol=1e-10)   # S_c by QR vs LU: the same determinant


def test_twin_qr_sign_convention():
    """det S_c = (-1)^reflections prod R_kk: with K = 0 every S_c = I (no reflection needed or taken), log det =
    n log s2; with a rank-1 kernel each coupling system has det > 0 (Sylvester); a sign error in the reflection
    count makes the twin report ENOTPD on these SPD matrices."""
    rng = np.random.default_rng(22)
    x = rng.uniform(0, 1, 512)
    t = OracleHODLR(x, SE, (0.0, 0.1), 1e-2, 16, 1e-12, twin=True).factor()
    assert t.logdet() == pytest.approx(512 * math.log(1e-2), rel=1e-14)
    t = OracleHODLR(x, SE, (1.0, 1e20), 1e-2, 16, 1e-12, twin=True).factor()
    assert t.logdet() == pytest.approx(511 * math.log(1e-2) + math.log(1e-2 + 512), rel=1e-13)


# ---------------------------------------------------------------------------------------------------------------
# NEXT-2: heteroscedastic noise C_ij = sigma_i^2 delta_ij + k(x_i, x_j)
def test_noise_zero_kernel_closed_form():
    """K = 0 with per-point noise: C = diag(s2 + noise_i), log det = sum log(s2 + noise_i), x = y / (s2 + noise_i)
    in the caller's order -- a noise vector applied in sorted instead of original order fails here."""
    rng = np.random.default_rng(31)
    n, s2 = 1000, 1e-3
    x = rng.uniform(0, 1, n); y = rng.standard_normal(n); nz = rng.uniform(0, 0.5, n)
    h = OracleHODLR(x, SE, (0.0, 0.1), s2, 32, 1e-12, noise=nz).factor()
    assert h.logdet() == pytest.approx(float(np.sum(np.log(s2 + nz))), rel=1e-13)
    np.testing.assert_allclose(h.solve(y), y / (s2 + nz), rtol=1e-14)


@pytest.mark.parametrize("kernel", [SE, MATERN32])
def test_noise_hodlr_vs_dense(kernel):
    """HODLR with heteroscedastic noise against numpy dense (independent assembly + LAPACK) and the O11 checker."""
    rng = np.random.default_rng(32 + kernel)
    n = 1500
    x = rng.uniform(0, 4, n); y = rng.standard_normal(n); nz = np.exp(rng.uniform(np.log(1e-4), np.log(1e-1), n))
    th = (1.0, 0.3)
    h = OracleHODLR(x, kernel, th, 0.0, 48, 1e-12, noise=nz).factor()
    C = dense_C(x, kernel, th, 0.0) + np.diag(nz)
    sd, ld = np.linalg.slogdet(C)
    assert sd > 0 and abs(h.logdet() - ld) <= 1e-12 * abs(ld)
    xd = np.linalg.solve(C, y)
    assert np.linalg.norm(h.solve(y) - xd) <= 1e-9 * np.linalg.norm(xd)
    ld2, x2 = dense_check(x, kernel, th, 0.0, y, noise=nz)
    assert abs(ld2 - ld) <= 1e-12 * abs(ld) and np.linalg.norm(x2 - xd) <= 1e-9 * np.linalg.norm(xd)
    with pytest.raises(OracleError):
        OracleHODLR(x, kernel, th, 0.0, 48, 1e-12, noise=-nz)


# ---------------------------------------------------------------------------------------------------------------
# NEXT-3 groundwork (oracle only): d-dimensional points with the kd-tree ordering of PAPER.md:666-677 (R19)
def _dense_C_nd(X, kernel, theta, s2):
    """Independent numpy assembly for d-dimensional points: Euclidean distances (scipy), Table I of r."""
    from scipy.spatial.distance import cdist
    r = cdist(X, X)
    a, ell = theta[0], theta[1]
    if kernel == SE:
        K = a * a * np.exp(-r * r / (2 * ell * ell))
    else:
        s = (3.0 ** 0.5 if kernel == MATERN32 else 5.0 ** 0.5) * r / ell
        K = a * a * ((1 + s) if kernel == MATERN32 else (1 + s + s * s / 3)) * np.exp(-s)
    return K + s2 * np.eye(len(X))


def test_kd_order_spec_square():
    """SPEC.md geometry example: the 2-D unit square with leaf size 1 -- the first split (on x) puts (0,0), (0,1)
    before (1,0), (1,1); the second level sorts each half by y."""
    X = np.array([[0.0, 0.0], [1.0, 0.0], [0.0, 1.0], [1.0, 1.0]])
    o = OracleHODLR(X, SE, (1.0, 1.0), 1e-2, 1, 1e-12)
    assert o.kappa == 2
    np.testing.assert_array_equal(o.perm(), [0, 2, 1, 3])
    np.testing.assert_array_equal(o.sorted_x(), X[[0, 2, 1, 3]])


@pytest.mark.parametrize("d", [2, 3])
def test_kd_order_invariants(d):
    """perm is a permutation; every internal node of depth L splits its points by coordinate L mod d (all of the
    left child's coordinates <= all of the right child's); ties in the split coordinate keep their relative
    order from the level above (checked by a plain re-implementation in Python: per-level stable sorts)."""
    rng = np.random.default_rng(40 + d)
    n = 1000
    X = np.round(rng.uniform(0, 4, (n, d)), 1)          # many ties
    o = OracleHODLR(X, SE, (1.0, 1.0), 1e-2, 16, 1e-12)
    p = o.perm()
    assert np.array_equal(np.sort(p), np.arange(n))
    lo, hi = o.tree()
    k = o.kappa
    Xs = X[p]
    for c in range((1 << k) - 1):
        L = int(np.floor(np.log2(c + 1)))
        cl, cr = 2 * c + 1, 2 * c + 2
        ax = L % d
        assert Xs[lo[cl]:hi[cl], ax].max() <= Xs[lo[cr]:hi[cr], ax].min()
    ref = np.arange(n)
    for L in range(k):
        for c in range((1 << L) - 1, (2 << L) - 1):
            seg = ref[lo[c]:hi[c]]
            ref[lo[c]:hi[c]] = seg[np.argsort(X[seg, L % d], kind="stable")]
    np.testing.assert_array_equal(p, ref)


def test_kd_order_one_dim_is_the_sort():
    """d = 1 given as an (n, 1) array: the same permutation and factorization as the 1-D input."""
    rng = np.random.default_rng(44)
    x = np.round(rng.uniform(0, 1, 777), 2); y = rng.standard_normal(777)
    a = OracleHODLR(x, MATERN32, (1.0, 0.2), 1e-2, 20, 1e-12).factor()
    b = OracleHODLR(x[:, None], MATERN32, (1.0, 0.2), 1e-2, 20, 1e-12).factor()
    np.testing.assert_array_equal(a.perm(), b.perm())
    assert a.logdet() == b.logdet()
    np.testing.assert_array_equal(a.solve(y), b.solve(y))


@pytest.mark.parametrize("d,kernel", [(2, SE), (2, MATERN32), (3, MATERN52)])
def test_kd_hodlr_vs_dense(d, kernel):
    """d-dimensional HODLR (kd ordering, Euclidean kernel entries) against numpy dense (scipy distances, LAPACK) and
    the O11 checker; a shuffled input gives the same log det."""
    rng = np.random.default_rng(50 + d + kernel)
    n = 1200
    X = rng.uniform(0, 1, (n, d)); y = rng.standard_normal(n)
    th = (1.0, 0.5)
    h = OracleHODLR(X, kernel, th, 1e-2, 32, 1e-12).factor()
    C = _dense_C_nd(X, kernel, th, 1e-2)
    sd, ld = np.linalg.slogdet(C)
    assert sd > 0 and abs(h.logdet() - ld) <= 1e-11 * abs(ld)
    xd = np.linalg.solve(C, y)
    assert np.linalg.norm(h.solve(y) - xd) <= 1e-8 * np.linalg.norm(xd)
    ld11, x11 = dense_check(X, kernel, th, 1e-2, y)
    assert abs(ld11 - ld) <= 1e-11 * abs(ld)
    q = rng.permutation(n)
    h2 = OracleHODLR(X[q], kernel, th, 1e-2, 32, 1e-12).factor()
    assert h2.logdet() == h.logdet()


# ---------------------------------------------------------------------------------------------------------------
# NEXT-2 (not positive definite): multiquadric (Table III) and biharmonic (Table VI), signed log det (R20)
from oracle import MQ, BIHARM  # noqa: E402


def test_nonspd_kernel_closed_forms():
    """MQ a^2 sqrt(1 + (d/ell)^2) and biharmonic a^2 (d/ell)^2 log|d/ell| at hand-checked points."""
    assert kernel_value(MQ, (2.0, 0.5), 0.5) == pytest.approx(4.0 * math.sqrt(2.0), rel=1e-15)
    assert kernel_value(MQ, (1.0, 1.0), 0.0) == 1.0
    assert kernel_value(BIHARM, (1.0, 1.0), math.e) == pytest.approx(math.e ** 2, rel=1e-15)
    assert kernel_value(BIHARM, (3.0, 2.0), 2.0) == 0.0           # log 1 = 0
    assert kernel_value(BIHARM, (1.0, 1.0), 0.0) == 0.0           # removable singularity
    assert kernel_value(BIHARM, (1.0, 1.0), -0.5) == pytest.approx(0.25 * math.log(0.5), rel=1e-15)


@pytest.mark.parametrize("kernel,s2,n", [(MQ, 1.0, 1500), (BIHARM, 2.0, 1500), (MQ, 1.0, 3000)])
def test_nonspd_hodlr_vs_dense(kernel, s2, n):
    """The paper's Table III / VI matrices C = s2 I + K on U[-3, 3] (1-D): HODLR (leaf LU, coupling systems of either
    sign) against numpy slogdet / LAPACK solve -- log |det| and sign -- and the unfactorable-as-covariance guard."""
    rng = np.random.default_rng(60 + kernel + n)
    x = rng.uniform(-3, 3, n); y = rng.standard_normal(n)
    d = np.abs(x[:, None] - x[None, :])
    if kernel == MQ:
        K = np.sqrt(1 + d * d)
    else:
        with np.errstate(divide="ignore", invalid="ignore"):
            K = np.where(d > 0, d * d * np.log(d), 0.0)
    Cm = K + s2 * np.eye(n)
    sd, ld = np.linalg.slogdet(Cm)
    h = OracleHODLR(x, kernel, (1.0, 1.0), s2, 64, 1e-12).factor()
    la, sg = h.logdet_sign()
    assert sg == int(sd) and abs(la - ld) <= 1e-11 * abs(ld)
    xs = h.solve(y)
    xd = np.linalg.solve(Cm, y)
    assert np.linalg.norm(xs - xd) <= 1e-8 * np.linalg.norm(xd)
    with pytest.raises(OracleError) as e:
        h.gp_loglik(y)
    assert e.value.status == "EINVAL"


def test_nonspd_sign_both_ways():
    """C = s2 I + MQ on U[-3, 3] has a handful of negative eigenvalues (7..10 here), so det C takes either sign with
    the shift: both signs and log |det| against numpy on well-conditioned cases (cond ~1e4)."""
    rng = np.random.default_rng(0)
    seen = set()
    for n, s2 in ((500, 1.0), (500, 0.5), (1000, 0.5), (1000, 1.0)):
        x = rng.uniform(-3, 3, n)
        d = np.abs(x[:, None] - x[None, :])
        sd, ld = np.linalg.slogdet(np.sqrt(1 + d * d) + s2 * np.eye(n))
        h = OracleHODLR(x, MQ, (1.0, 1.0), s2, 32, 1e-12).factor()
        la, sg = h.logdet_sign()
        assert sg == int(sd) and abs(la - ld) <= 1e-11 * abs(ld), (n, s2)
        seen.add(sg)
    assert seen == {1, -1}


def test_points_nd_recipe():
    """NEXT-3 input recipe: seeded, inside the cube, y drawn after x; the lattice option gives
    exact coordinate ties and duplicate points (the cases the kd sort's tie rule and the duplicate-row rule cover)."""
    from paper_1403_6015_b200 import inputs
    x, y = inputs.points_nd(5000, 3, seed=7, half=0.5)
    x2, y2 = inputs.points_nd(5000, 3, seed=7, half=0.5)
    assert x.shape == (5000, 3) and y.shape == (5000,)
    np.testing.assert_array_equal(x, x2); np.testing.assert_array_equal(y, y2)
    assert np.all(np.abs(x) <= 0.5)
    g, _ = inputs.points_nd(6000, 2, seed=3, half=0.5, grid=16)
    assert len(np.unique(g[:, 0])) <= 17
    assert len(np.unique(g, axis=0)) < len(g)
