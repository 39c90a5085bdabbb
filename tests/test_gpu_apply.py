"""GPU parity of the forward apply Y = C~ X (NEXT-1 of SURVEY 8(f), include/hodlr.h hodlr_apply) through the C-ABI
against the oracle's apply (oracle/hodlr_oracle.c oracle_apply: leaf blocks dense + U V^T of every ACA block).

Both sides apply the operator of their own ACA factors; these agree to the compression tolerance (ranks may differ
by <= 2 in a few blocks, R11), so the gate is relative to eps: ||y_gpu - y_oracle|| <= 100 eps ||y||
(eps = 1e-12: 1e-10).  apply(solve(y)) = y checks that the solve inverts exactly the operator applied
(to rounding x cond(C)).
"""
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


def _cases():
    c1 = inputs.CONFIGS["cfg1"]
    c2 = inputs.CONFIGS["cfg2"]
    c3 = inputs.scaled(inputs.CONFIGS["cfg3"], 1 << 15)
    c5 = inputs.scaled(inputs.CONFIGS["cfg5"], 1 << 14)          # clustered duplicates
    return [("cfg1", c1, c1.eps), ("cfg2", c2, c2.eps), ("cfg3@2^15", c3, c3.eps), ("cfg5@2^14", c5, c5.eps)]


@pytest.mark.parametrize("name,cfg,eps", _cases(), ids=[c[0] for c in _cases()])
def test_apply_matches_oracle(hb, name, cfg, eps):
    x = inputs.points(cfg)
    n = x.size
    rng = np.random.default_rng(7)
    V = rng.standard_normal((n, 2))
    o = OracleHODLR(x, cfg.kernel, cfg.theta, cfg.sigma2, cfg.leaf, eps)
    Yo = np.stack([o.apply(V[:, j]) for j in range(2)], axis=1)
    g = hb.HODLR(torch.from_numpy(x).cuda(), cfg.kernel, cfg.theta, cfg.sigma2, cfg.leaf, eps)
    Yg = g.apply(torch.from_numpy(V).cuda()).cpu().numpy()          # before factor: legal
    rel = np.linalg.norm(Yg - Yo) / np.linalg.norm(Yo)
    print(f"[apply] {name} n={n} rel {rel:.2e}")
    assert rel <= max(100 * eps, 1e-12), rel
    y1 = g.apply(torch.from_numpy(V[:, 0].copy()).cuda()).cpu().numpy()
    np.testing.assert_array_equal(y1, Yg[:, 0])                        # 1-column call = column 0, bitwise
    g.close()


@pytest.mark.parametrize("name,cfg,eps", _cases()[:3], ids=[c[0] for c in _cases()[:3]])
def test_apply_inverts_solve(hb, name, cfg, eps):
    x = inputs.points(cfg); y = inputs.rhs(cfg)
    g = hb.HODLR(torch.from_numpy(x).cuda(), cfg.kernel, cfg.theta, cfg.sigma2, cfg.leaf, eps).factor()
    yd = torch.from_numpy(y).cuda()
    r = g.apply(g.solve(yd)) - yd
    rel = (torch.linalg.norm(r) / torch.linalg.norm(yd)).item()
    print(f"[apply] {name} ||apply(solve(y)) - y|| / ||y|| = {rel:.2e}")
    assert rel <= 2e-10, rel                # ~cond(C) x 1e-16 at these configs (cfg2: 1.2e-10)
    g.close()


def test_apply_small_and_ragged(hb):
    for n, leaf in ((1, 16), (17, 16), (64, 64), (3001, 37)):
        cfg = inputs.scaled(inputs.CONFIGS["cfg1"], n)
        x = inputs.points(cfg)
        v = np.random.default_rng(n).standard_normal(n)
        o = OracleHODLR(x, cfg.kernel, cfg.theta, cfg.sigma2, leaf, 1e-12)
        yo = o.apply(v)
        g = hb.HODLR(torch.from_numpy(x).cuda(), cfg.kernel, cfg.theta, cfg.sigma2, leaf, 1e-12)
        yg = g.apply(torch.from_numpy(v).cuda()).cpu().numpy()
        assert np.linalg.norm(yg - yo) <= 1e-10 * np.linalg.norm(yo), (n, leaf)
        g.close()


def test_apply_errors(hb):
    cfg = inputs.CONFIGS["cfg1"]
    x = torch.from_numpy(inputs.points(cfg)).cuda()
    g = hb.HODLR(x, cfg.kernel, cfg.theta, cfg.sigma2, cfg.leaf, cfg.eps)
    lib = hb.load()
    v = torch.zeros(cfg.n, dtype=torch.float64, device="cuda")
    out = torch.empty_like(v)
    assert lib.hodlr_apply(g._h, v.data_ptr(), out.data_ptr(), 0, cfg.n) == 1          # nrhs < 1
    assert lib.hodlr_apply(g._h, v.data_ptr(), out.data_ptr(), 1, cfg.n - 1) == 1      # ld < n
    assert lib.hodlr_apply(g._h, None, out.data_ptr(), 1, cfg.n) == 1                  # NULL
    g.close()
