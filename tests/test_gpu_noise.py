"""NEXT-2 heteroscedastic noise C_ij = sigma_i^2 delta_ij + k(x_i, x_j) (hodlr_opts.noise):
GPU against the oracle, through the C-ABI."""
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


@pytest.mark.parametrize("name,n", [("cfg1", 2048), ("cfg2", 1 << 14), ("cfg3", 1 << 15)])
def test_noise_parity(hb, name, n):
    cfg = inputs.scaled(inputs.CONFIGS[name], n)
    x = inputs.points(cfg, sort=False); y = inputs.rhs(cfg)
    nz = np.exp(np.random.default_rng(77).uniform(np.log(1e-4), np.log(1e-1), n))
    o = OracleHODLR(x, cfg.kernel, cfg.theta, cfg.sigma2, cfg.leaf, 1e-12, noise=nz).factor()
    ld_o = o.logdet(); x_o = o.solve(y)
    g = hb.HODLR(torch.from_numpy(x).cuda(), cfg.kernel, cfg.theta, cfg.sigma2, cfg.leaf, 1e-12,
                 noise=torch.from_numpy(nz).cuda())
    xg, quad = g.factor_solve(torch.from_numpy(y).cuda())
    xg = xg.cpu().numpy()
    assert abs(g.logdet() - ld_o) <= 1e-9 * abs(ld_o)
    assert np.linalg.norm(xg - x_o) <= 1e-9 * np.linalg.norm(x_o)
    assert abs(quad - y @ x_o) <= 1e-9 * abs(y @ x_o)
    ya = torch.from_numpy(np.sin(x)).cuda()            # the forward apply carries the same diagonal
    assert np.linalg.norm(g.apply(ya).cpu().numpy() - o.apply(np.sin(x))) <= 1e-12 * np.linalg.norm(o.apply(np.sin(x)))


def test_noise_errors(hb):
    xd = torch.linspace(0, 1, 300, dtype=torch.float64, device="cuda")
    bad = torch.full((300,), 0.1, dtype=torch.float64, device="cuda"); bad[17] = -1.0
    with pytest.raises(hb.HodlrError) as e:
        hb.HODLR(xd, 0, (1.0, 0.1), 1e-2, 32, 1e-12, noise=bad)
    assert e.value.status == "EINVAL"
    bad[17] = float("nan")
    with pytest.raises(hb.HodlrError) as e:
        hb.HODLR(xd, 0, (1.0, 0.1), 1e-2, 32, 1e-12, noise=bad)
    assert e.value.status == "EINVAL"
