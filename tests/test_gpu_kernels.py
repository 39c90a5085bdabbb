"""GPU parity for the NEXT-2 covariance functions (include/hodlr.h: EXP = Ornstein-Uhlenbeck, Table I / Table IV;
IMQ = inverse multiquadric, Table V; RQ = rational quadratic, Table I) through the C-ABI against the oracle,
at eps = 1e-12 with the north_star gates (log det / log-likelihood 1e-9, solve 1e-9, structures bit-exact)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import EXP, IMQ, RQ  # noqa: E402
from test_gpu_parity import run_both, check_parity  # noqa: E402


@pytest.fixture(scope="module")
def hb():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1403_6015_b200.hodlr as hb
    hb.load()
    return hb


CASES = [
    ("exp", 16384, 0.0, 40.0, EXP, (1.1, 0.5), 1e-2, 64),
    ("imq", 8192, -3.0, 3.0, IMQ, (1.0, 0.05), 1e-1, 64),
    ("rq", 8192, 0.0, 20.0, RQ, (0.9, 0.4, 1.5), 1e-2, 128),
    ("rq-ragged", 3001, 0.0, 7.0, RQ, (1.0, 0.3, 0.7), 1e-2, 37),
]


@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_next2_kernel_parity(hb, case):
    _, n, lo, hi, k, th, s2, leaf = case
    rng = np.random.default_rng(5)
    x = np.sort(rng.uniform(lo, hi, n)); y = rng.standard_normal(n)
    o, g, ro, rg = run_both(hb, x, y, k, th, s2, leaf, 1e-12)
    check_parity(o, g, ro, rg)
    g.close()


def test_rq_needs_alpha(hb):
    x = torch.linspace(0, 1, 100, dtype=torch.float64, device="cuda")
    with pytest.raises(hb.HodlrError):
        hb.HODLR(x, RQ, (1.0, 0.5, 0.0), 1e-2, 16, 1e-10)
