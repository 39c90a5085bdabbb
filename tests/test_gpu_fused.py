"""hodlr_factor_solve: the right-hand side fused into the factorization against the oracle, and
against the unfused path on the same handle shape.  Through the C-ABI (ctypes binding)."""
import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import OracleHODLR  # noqa: E402
from paper_1403_6015_b200 import inputs  # noqa: E402

TOL = 1e-9


@pytest.fixture(scope="module")
def hb():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1403_6015_b200.hodlr as hb
    hb.load()
    return hb


def fused_vs_oracle(hb, x, y, kernel, theta, s2, leaf, eps=1e-12, dist=None):
    o = OracleHODLR(x, kernel, theta, s2, leaf, eps).factor()
    ld_o = o.logdet(); x_o = o.solve(y)
    quad_o = float(y @ x_o)
    g = hb.HODLR(torch.from_numpy(x).cuda(), kernel, theta, s2, leaf, eps, dist=dist)
    xg, quad = g.factor_solve(torch.from_numpy(y).cuda())
    xg = xg.cpu().numpy()
    ld_g = g.logdet()
    rel = np.linalg.norm(xg - x_o) / np.linalg.norm(x_o)
    print(f"[fused n={x.size}] logdet rel {abs(ld_g - ld_o) / abs(ld_o):.2e} solve rel {rel:.2e} "
          f"quad rel {abs(quad - quad_o) / abs(quad_o):.2e}")
    assert abs(ld_g - ld_o) <= TOL * abs(ld_o) + 1e-12
    assert rel <= TOL
    assert abs(quad - quad_o) <= TOL * abs(quad_o) + 1e-12
    return o, g


@pytest.mark.parametrize("name,n", [("cfg1", 2048), ("cfg2", 65536), ("cfg3", 1 << 16), ("cfg5", 1 << 15)])
def test_fused_configs(hb, name, n):
    cfg = inputs.scaled(inputs.CONFIGS[name], n)
    x = inputs.points(cfg); y = inputs.rhs(cfg)
    o, g = fused_vs_oracle(hb, x, y, cfg.kernel, cfg.theta, cfg.sigma2, cfg.leaf)
    # the handle is factored: a second right-hand side through the ordinary solve, and the log-likelihood
    y2 = np.cos(np.arange(n) * 0.37)
    x2 = g.solve(torch.from_numpy(y2).cuda()).cpu().numpy()
    x2o = o.solve(y2)
    assert np.linalg.norm(x2 - x2o) <= TOL * np.linalg.norm(x2o)
    ll = g.gp_loglik(torch.from_numpy(y).cuda())
    assert abs(ll - o.gp_loglik(y)) <= TOL * (abs(o.gp_loglik(y)) + abs(o.logdet()))


@pytest.mark.parametrize("n,leaf", [(1, 64), (17, 64), (64, 64), (128, 64), (1999, 50), (3001, 37), (4097, 128)])
def test_fused_edge_sizes(hb, n, leaf):
    rng = np.random.default_rng(100 + n)
    x = rng.uniform(-3, 3, n); y = rng.standard_normal(n)
    fused_vs_oracle(hb, x, y, 0, (1.0, 1 / math.sqrt(2)), 1.0, leaf)


@pytest.mark.parametrize("kernel", [1, 2])
def test_fused_unsorted_matern(hb, kernel):
    rng = np.random.default_rng(9 + kernel)
    x = np.round(rng.uniform(0, 20, 5000), 2); y = rng.standard_normal(5000)
    fused_vs_oracle(hb, x, y, kernel, (1.3, 0.7), 1e-2, 64)


def test_fused_quad_only_and_errors(hb):
    cfg = inputs.CONFIGS["cfg1"]
    x = inputs.points(cfg); y = inputs.rhs(cfg)
    g = hb.HODLR(torch.from_numpy(x).cuda(), cfg.kernel, cfg.theta, cfg.sigma2, cfg.leaf, 1e-12)
    xs, quad = g.factor_solve(torch.from_numpy(y).cuda(), solve=False)
    assert xs is None
    o = OracleHODLR(x, cfg.kernel, cfg.theta, cfg.sigma2, cfg.leaf, 1e-12).factor()
    assert abs(quad - y @ o.solve(y)) <= TOL * abs(quad)
    with pytest.raises(hb.HodlrError) as e:          # already factored
        g.factor_solve(torch.from_numpy(y).cuda())
    assert e.value.status == "ESTATE"
    yb = y.copy(); yb[5] = np.nan
    g2 = hb.HODLR(torch.from_numpy(x).cuda(), cfg.kernel, cfg.theta, cfg.sigma2, cfg.leaf, 1e-12)
    with pytest.raises(hb.HodlrError) as e:
        g2.factor_solve(torch.from_numpy(yb).cuda())
    assert e.value.status == "EINVAL"
    assert abs(g2.logdet() - o.logdet()) <= TOL * abs(o.logdet())   # the factorization itself is valid


def test_factor_solve_into_pinned_host(hb):
    """x of hodlr_factor_solve in page-locked host memory (written by the solve kernel through the unified address)
    equals the device result bit for bit; pageable host memory is refused (include/hodlr.h)."""
    import numpy as np
    rng = np.random.default_rng(11)
    n = 20000
    x = torch.from_numpy(np.sort(rng.uniform(0, 50, n))).cuda()
    y = torch.from_numpy(rng.standard_normal(n)).cuda()
    g = hb.HODLR(x, 0, (1.0, 1.0), 1e-2, 128, 1e-10)
    sd, qd = g.factor_solve(y)
    g.close()
    pin = torch.empty(n, dtype=torch.float64).pin_memory()
    g = hb.HODLR(x, 0, (1.0, 1.0), 1e-2, 128, 1e-10)
    sp, qp = g.factor_solve(y, out=pin)
    g.close()
    assert sp.data_ptr() == pin.data_ptr() and qp == qd
    assert torch.equal(pin, sd.cpu())
    g = hb.HODLR(x, 0, (1.0, 1.0), 1e-2, 128, 1e-10)
    with pytest.raises(TypeError):
        g.factor_solve(y, out=torch.empty(n, dtype=torch.float64))          # pageable: refused by the binding
    arr = np.zeros(n)                                                       # ... and by the C-ABI (HODLR_EINVAL)
    assert hb.load().hodlr_factor_solve(g._h, y.data_ptr(), arr.ctypes.data, None) == 1
    g.close()
