"""Size-independent properties at the full BASELINE sizes, where the oracle
cannot follow the whole run: linearity of the integrator (M x'' + K x = 0 is
linear and every RK4 stage is a linear map, so a mix of runs equals the run of
the mix to rounding), an approximate time-reversal round trip, and the
reference's energy-drift bound (test_acceptance.py:115-120, drift < 1e-6)."""

import numpy as np
import pytest

from paper_1702_02207_b200 import workloads

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_1702_02207_b200 import batched  # noqa: E402


def _lin_check(run, x0, v0, y0, w0, alpha=0.7, beta=-1.3):
    a = run(x0, v0)
    b = run(y0, w0)
    mix = run(alpha * x0 + beta * y0, alpha * v0 + beta * w0)
    for got, p, q in ((mix.x, a.x, b.x), (mix.v, a.v, b.v)):
        expect = alpha * p + beta * q
        err = (got - expect).abs() / expect.abs().clamp_min(1.0)
        assert float(err.max()) <= 1e-9


def test_linearity_c2_full_size():
    m, C, x0, v0 = workloads.c2()
    rng = np.random.default_rng(1)
    y0, w0 = rng.standard_normal(x0.shape), rng.standard_normal(x0.shape)
    v0 = rng.standard_normal(x0.shape)
    dev = lambda a: torch.from_numpy(a).cuda()  # noqa: E731
    m, C = dev(m), dev(C)
    _lin_check(lambda x, v: batched.integrate_batch2(m, C, x, v, 1e-4, 10_000),
               dev(x0), dev(v0), dev(y0), dev(w0))


def test_linearity_c3_full_chain():
    m, C, x0, v0 = workloads.c3()
    rng = np.random.default_rng(2)
    y0 = rng.standard_normal(x0.shape)
    dev = lambda a: torch.from_numpy(a).cuda()  # noqa: E731
    m, C = dev(m), dev(C)
    zero = torch.zeros_like(m)
    _lin_check(lambda x, v: batched.integrate_chains(m, C, x, v, 1e-4, 2000), dev(x0), zero,
               dev(y0), zero)


def test_reversal_c4_full_size():
    """Integrate forward, negate velocities, integrate back: returns within the
    reference's 1e-6 bound (RK4 is not exactly time-symmetric)."""
    m, C, x0, v0 = workloads.c4()
    fwd = batched.integrate_chains(m, C, x0, v0, 1e-4, 2000)
    back = batched.integrate_chains(m, C, fwd.x, -fwd.v, 1e-4, 2000)
    assert float((back.x - torch.from_numpy(x0).cuda()).abs().max()) < 1e-6


def test_energy_drift_c4_full_size():
    m, C, x0, v0 = workloads.c4()
    res = batched.integrate_chains(m, C, x0, v0, 1e-4, 10_000, 2000, energies=True)
    d = res.energy_drift().cpu().numpy()
    assert np.isfinite(d).all() and d.max() < 1e-6
