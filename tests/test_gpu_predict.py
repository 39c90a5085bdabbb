"""GPU parity of GP prediction (NEXT-1, include/hodlr.h gp_predict; eq_reg1 / eq_reg2) against
the oracle's predict (its own HODLR solve + entry-wise cross-covariances), and the sec. 5.6 regression experiment
(PAPER.md:1656-1705): |RMSE(HODLR) - RMSE(dense)| shrinks in proportion to eps.

Gates: mean ||d|| / ||mean|| <= 1e-9 and |d var| <= 1e-9 a^2 at eps = 1e-12 (both sides solve with their own ACA
factors, equal to the compression tolerance).
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import OracleHODLR, SE  # noqa: E402
from paper_1403_6015_b200 import inputs  # noqa: E402


@pytest.fixture(scope="module")
def hb():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1403_6015_b200.hodlr as hb
    hb.load()
    return hb


@pytest.mark.parametrize("name,n", [("cfg1", 2048), ("cfg2", 1 << 13)])
def test_predict_matches_oracle(hb, name, n):
    cfg = inputs.scaled(inputs.CONFIGS[name], n)
    x = inputs.points(cfg, sort=False); y = inputs.rhs(cfg)
    rng = np.random.default_rng(3)
    xt = rng.uniform(cfg.lo - 0.05 * (cfg.hi - cfg.lo), cfg.hi + 0.05 * (cfg.hi - cfg.lo), 40)
    o = OracleHODLR(x, cfg.kernel, cfg.theta, cfg.sigma2, cfg.leaf, 1e-12).factor()
    mo, vo = o.predict(y, xt)
    g = hb.HODLR(torch.from_numpy(x).cuda(), cfg.kernel, cfg.theta, cfg.sigma2, cfg.leaf, 1e-12).factor()
    mg, vg = g.predict(torch.from_numpy(y).cuda(), torch.from_numpy(xt).cuda())
    mg = mg.cpu().numpy(); vg = vg.cpu().numpy()
    rel = np.linalg.norm(mg - mo) / np.linalg.norm(mo)
    dv = np.max(np.abs(vg - vo))
    print(f"[predict] {name} n={n} mean rel {rel:.2e} var max abs {dv:.2e}")
    assert rel <= 1e-9, rel
    assert dv <= 1e-9 * cfg.a ** 2, dv
    m2, v2 = g.predict(torch.from_numpy(y).cuda(), torch.from_numpy(xt).cuda(), variance=False)
    assert v2 is None
    np.testing.assert_array_equal(m2.cpu().numpy(), mg)               # mean does not depend on the variance pass
    g.close()


def test_rmse_experiment_sec_5_6(hb):
    """sec. 5.6: y_hat = K (sigma^2 I + K)^{-1} y at the data points, k = exp(-(x - x')^2) (a = 1, ell = 1/sqrt 2),
    sigma_eps = 1, p_max = 20, 1024 points.  y_hat = y - sigma^2 alpha with alpha from the HODLR solve (and, as a
    cross-check, the predictive mean at the data points); RMSE = ||y - y_hat|| / sqrt(1024)."""
    x, y = inputs.rmse_model()
    theta, s2, leaf = (1.0, 1.0 / np.sqrt(2.0)), 1.0, 20
    d = x[:, None] - x[None, :]
    K = np.exp(-d * d)
    yhat_exact = K @ np.linalg.solve(K + s2 * np.eye(x.size), y)
    rmse_exact = np.linalg.norm(y - yhat_exact) / np.sqrt(x.size)
    assert 0.8 < rmse_exact < 1.2, rmse_exact                        # noise level sigma_eps = 1
    xd = torch.from_numpy(x).cuda(); yd = torch.from_numpy(y).cuda()
    diffs = {}
    for eps in (1e-3, 1e-5, 1e-7, 1e-9, 1e-11):
        g = hb.HODLR(xd, SE, theta, s2, leaf, eps).factor()
        alpha = g.solve(yd)
        yhat = (yd - s2 * alpha).cpu().numpy()
        mean, _ = g.predict(yd, xd, variance=False)
        np.testing.assert_allclose(mean.cpu().numpy(), yhat, rtol=0, atol=1e-9 * np.abs(yhat).max() + 1e3 * eps)
        rmse = np.linalg.norm(y - yhat) / np.sqrt(x.size)
        diffs[eps] = abs(rmse - rmse_exact)
        g.close()
    print("[rmse] exact", rmse_exact, {f"{e:.0e}": f"{v:.1e}" for e, v in diffs.items()})
    for eps, dv in diffs.items():
        assert dv <= 10 * eps, (eps, dv)                              # |d RMSE| proportional to eps (Fig. 9)
