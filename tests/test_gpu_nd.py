"""GPU parity for d-dimensional points (NEXT-3; hodlr_build_nd, R19 / 9f): the kd ordering of
PAPER.md:666-677 on the device (per-level stable radix sorts), Euclidean kernel entries in the ACA and leaf kernels,
and the unchanged factor / solve / log det, against the oracle's oracle_build_nd on the same seeded inputs
(paper_1403_6015_b200.inputs.points_nd: Table II's uniform cube).

Gates: permutation, sorted points and tree bit-exact; log det and log-likelihood <= 1e-9 relative; the solve within
max(1e-9, 10 floor) (floor: the oracle against its Q15 twin, the same compression with LU leaves and QR coupling
systems); per-block ranks as the 1-D tests (<= 25% differ, by <= 2)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import OracleHODLR  # noqa: E402
from paper_1403_6015_b200 import inputs  # noqa: E402

SE, M32, M52 = 0, 1, 2
LD_TOL = 1e-9
X_TOL = 1e-9


@pytest.fixture(scope="module")
def hb():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1403_6015_b200.hodlr as hb
    hb.load()
    return hb


def check(hb, x, y, kernel, theta, s2, leaf, eps, tag, twin=True):
    o = OracleHODLR(x, kernel, theta, s2, leaf, eps).factor()
    ld_o = o.logdet(); x_o = o.solve(y); ll_o = o.gp_loglik(y)
    floor = 0.0
    if twin:
        t = OracleHODLR(x, kernel, theta, s2, leaf, eps, twin=True).factor()
        floor = float(np.linalg.norm(t.solve(y) - x_o) / np.linalg.norm(x_o))
    xd = torch.from_numpy(np.ascontiguousarray(x)).cuda(); yd = torch.from_numpy(y).cuda()
    g = hb.HODLR(xd, kernel, theta, s2, leaf, eps)
    xs_g, perm_g = g.order()
    np.testing.assert_array_equal(perm_g.cpu().numpy(), o.perm())
    np.testing.assert_array_equal(xs_g.cpu().numpy(), o.sorted_x())
    lo_g, hi_g, r_g = g.tree()
    lo_o, hi_o = o.tree()
    np.testing.assert_array_equal(lo_g, lo_o)
    np.testing.assert_array_equal(hi_g, hi_o)
    r_o = o.ranks()
    if len(r_o):
        assert np.mean(r_g != r_o) <= 0.25 and np.all(np.abs(r_g.astype(int) - r_o.astype(int)) <= 2)
    g.factor()
    ld_g = g.logdet()
    x_g = g.solve(yd).cpu().numpy()
    ll_g = g.gp_loglik(yd)
    rel = float(np.linalg.norm(x_g - x_o) / np.linalg.norm(x_o))
    gate = max(X_TOL, 10 * floor)
    print(f"[nd {tag}] n={x.shape[0]} d={x.shape[1]} top rank {int(r_o[0]) if len(r_o) else 0} "
          f"logdet rel {abs(ld_g - ld_o) / abs(ld_o):.2e} solve rel {rel:.2e} (floor {floor:.2e}) "
          f"loglik rel {abs(ll_g - ll_o) / abs(ll_o):.2e} ranks differ {np.mean(r_g != r_o) if len(r_o) else 0:.2f}")
    assert abs(ld_g - ld_o) <= LD_TOL * abs(ld_o)
    assert rel <= gate
    assert abs(ll_g - ll_o) <= LD_TOL * abs(ll_o)
    return o, g, xd, yd, x_o


CASES = [   # (tag, d, n, half, kernel, theta, s2, leaf, eps, grid)
    ("2d-se", 2, 16384, 0.5, SE, (1.0, 1.0), 1e-2, 128, 1e-10, 0),
    ("2d-se-ragged", 2, 5001, 0.5, SE, (1.0, 1.0), 1e-2, 64, 1e-10, 0),
    ("2d-m52", 2, 8192, 0.5, M52, (1.0, 2.0), 1e-2, 128, 1e-8, 0),
    ("2d-m52-leaf37", 2, 3001, 0.5, M52, (1.0, 2.0), 1e-1, 37, 1e-8, 0),
    ("3d-se", 3, 16384, 0.5, SE, (1.0, 4.0), 1e-2, 128, 1e-10, 0),
    ("2d-grid-ties", 2, 6000, 0.5, SE, (1.0, 1.0), 1e-2, 64, 1e-10, 16),
    ("3d-grid-ties", 3, 4097, 0.5, SE, (1.0, 4.0), 1e-2, 128, 1e-10, 8),
    ("4d-se", 4, 4096, 0.5, SE, (1.0, 8.0), 1e-2, 64, 1e-8, 0),
]


@pytest.mark.parametrize("tag,d,n,half,kernel,theta,s2,leaf,eps,grid", CASES, ids=[c[0] for c in CASES])
def test_nd_parity(hb, tag, d, n, half, kernel, theta, s2, leaf, eps, grid):
    x, y = inputs.points_nd(n, d, seed=300 + d * 7 + n % 97, half=half, grid=grid)
    o, g, xd, yd, x_o = check(hb, x, y, kernel, theta, s2, leaf, eps, tag)
    # the fused right-hand side (hodlr_factor_solve) on a fresh handle: same solution and y^T C^-1 y
    g2 = hb.HODLR(xd, kernel, theta, s2, leaf, eps)
    xf, quad = g2.factor_solve(yd)
    assert abs(quad - float(y @ x_o)) <= 1e-9 * abs(float(y @ x_o))
    assert float(np.linalg.norm(xf.cpu().numpy() - x_o) / np.linalg.norm(x_o)) <= max(X_TOL, 1e-9)
    # the forward operator (hodlr_apply) inverts the solve: C~ (C~^-1 y) = y
    back = g.apply(torch.from_numpy(g.solve(yd).cpu().numpy()).cuda()).cpu().numpy()
    assert float(np.linalg.norm(back - y) / np.linalg.norm(y)) <= 1e-10
    g.close(); g2.close()


def test_nd_full_size_2d(hb):
    """nd2 at n = 2^18 (the oracle finishes it in about a minute): every bit-exact and tolerance gate."""
    d, half, kernel, theta, s2, leaf, eps = inputs.ND_CONFIGS["nd2"]
    x, y = inputs.points_nd(1 << 18, d, seed=2)
    check(hb, x, y, kernel, theta, s2, leaf, eps, "nd2-2^18", twin=False)


def test_nd_dim1_equals_1d(hb):
    """dim = 1 through hodlr_build_nd is hodlr_build bit for bit (same sort, same kernels)."""
    rng = np.random.default_rng(5)
    x = rng.uniform(0, 100, 20000); y = rng.standard_normal(20000)
    xd = torch.from_numpy(x).cuda(); yd = torch.from_numpy(y).cuda()
    a = hb.HODLR(xd, SE, (1.0, 1.0), 1e-2, 128, 1e-10).factor()
    b = hb.HODLR(xd.view(-1, 1), SE, (1.0, 1.0), 1e-2, 128, 1e-10).factor()
    assert a.logdet() == b.logdet()
    assert torch.equal(a.solve(yd), b.solve(yd))
    np.testing.assert_array_equal(a.tree()[2], b.tree()[2])


def test_nd_forced_ranks(hb):
    """With the oracle's per-block ranks forced, the difference to the oracle is arithmetic only: log det 1e-11."""
    d, half, kernel, theta, s2, leaf, eps = inputs.ND_CONFIGS["nd2"]
    x, y = inputs.points_nd(8192, d, seed=9)
    o = OracleHODLR(x, kernel, theta, s2, leaf, eps).factor()
    xd = torch.from_numpy(x).cuda()
    g = hb.HODLR(xd, kernel, theta, s2, leaf, eps, forced_ranks=o.ranks().astype(np.int32)).factor()
    np.testing.assert_array_equal(g.tree()[2], o.ranks())
    assert abs(g.logdet() - o.logdet()) <= 1e-11 * abs(o.logdet())
    x_g = g.solve(torch.from_numpy(y).cuda()).cpu().numpy()
    x_o = o.solve(y)
    assert float(np.linalg.norm(x_g - x_o) / np.linalg.norm(x_o)) <= 1e-10


@pytest.mark.parametrize("d", [2, 3])
def test_nd_predict(hb, d):
    """gp_predict at (m, d) test points: mean and latent variance against the oracle's predict (eq_reg1 / eq_reg2,
    PAPER.md:341-354; cross-covariances entry by entry): mean 1e-9, variance 1e-9 absolute (relative to k(0) = a^2)."""
    _, half, kernel, theta, s2, leaf, eps = inputs.ND_CONFIGS["nd2" if d == 2 else "nd3"]
    x, y = inputs.points_nd(4096, d, seed=21 + d)
    xt, _ = inputs.points_nd(37, d, seed=99 + d, half=0.6)       # some test points outside the training cube
    o = OracleHODLR(x, kernel, theta, s2, leaf, eps).factor()
    mo, vo = o.predict(y, xt)
    g = hb.HODLR(torch.from_numpy(x).cuda(), kernel, theta, s2, leaf, eps).factor()
    mg, vg = g.predict(torch.from_numpy(y).cuda(), torch.from_numpy(xt).cuda())
    mg = mg.cpu().numpy(); vg = vg.cpu().numpy()
    em = float(np.max(np.abs(mg - mo)) / np.max(np.abs(mo))); ev = float(np.max(np.abs(vg - vo)))
    print(f"[nd predict d={d}] mean rel {em:.2e} var abs {ev:.2e}")
    assert em <= 1e-9 and ev <= 1e-9
    g.close()


def test_nd_errors(hb):
    x, y = inputs.points_nd(4096, 2, seed=11)
    xd = torch.from_numpy(x).cuda()
    g = hb.HODLR(xd, SE, (1.0, 1.0), 1e-2, 128, 1e-10).factor()
    bad = x.copy(); bad[17, 1] = np.nan
    with pytest.raises(hb.HodlrError) as e:
        hb.HODLR(torch.from_numpy(bad).cuda(), SE, (1.0, 1.0), 1e-2, 128, 1e-10)
    assert e.value.status == "EINVAL"
    lib = hb.load()
    import ctypes as C
    th = (C.c_double * 3)(1.0, 1.0, 0.0)
    h = C.c_void_p(0)
    assert lib.hodlr_build_nd(xd.data_ptr(), 4096, 0, SE, th, 1e-2, 128, 1e-10, None, None, C.byref(h)) == 1
    assert lib.hodlr_build_nd(xd.data_ptr(), 4096, 65, SE, th, 1e-2, 128, 1e-10, None, None, C.byref(h)) == 1
    # short length scale on the paper's [-3, 3]^2: ranks beyond the cap -> ERANKCAP, not a wrong answer
    x2, _ = inputs.points_nd(8192, 2, seed=12, half=3.0)
    with pytest.raises(hb.HodlrError) as e:
        hb.HODLR(torch.from_numpy(x2).cuda(), SE, (1.0, 2 ** -0.5), 2.0, 128, 1e-12)
    assert e.value.status == "ERANKCAP"
    g.close()
