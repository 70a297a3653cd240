"""Property-based parity of the GPU path against the C oracle (which is
pinned to the reference in tests/test_oracle.py): random batches and chains,
random step counts, strides, tile depths and step sizes (stable and
diverging), with +-0, subnormal, tiny and huge entries.  Bar: byte-equal
samples and final states, equal first divergence steps."""

import numpy as np
import pytest
from hypothesis import HealthCheck, event, given, settings, strategies as st

import oracle
from conftest import bits

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_1702_02207_b200 import batched  # noqa: E402

SETTINGS = settings(max_examples=200, deadline=None,
                    suppress_health_check=[HealthCheck.too_slow, HealthCheck.data_too_large])
DT = st.sampled_from([1e-5, 1e-4, 1e-3, 5e-3, 2e-2, 0.3])


def _draw_state(rng, shape, special):
    m = rng.uniform(0.3, 3.0, shape) * 10.0 ** rng.integers(-2, 3, shape)
    C = rng.uniform(100.0, 3000.0, shape)
    x0 = rng.standard_normal(shape) * 10.0 ** rng.integers(-3, 4, shape)
    v0 = rng.standard_normal(shape) * rng.choice([0.0, 1.0, 100.0], shape)
    if special:
        flat = [a.reshape(-1) for a in (x0, v0)]
        n = flat[0].size
        for a in flat:
            k = rng.integers(0, n, max(1, n // 20))
            a[k] = rng.choice([0.0, -0.0, 5e-324, 1e-310, 1e-200, 1e150], k.size)
    return m, C, x0, v0


@SETTINGS
@given(B=st.integers(1, 3000), nsteps=st.integers(1, 300), sdiv=st.integers(1, 8),
       dt=DT, seed=st.integers(0, 2**32 - 1), special=st.booleans())
def test_batch2_random(B, nsteps, sdiv, dt, seed, special):
    rng = np.random.default_rng(seed)
    m, C, x0, v0 = _draw_state(rng, (2, B), special)
    stride = max(1, nsteps // sdiv + (seed % 3))
    res = batched.integrate_batch2(m, C, x0, v0, dt, nsteps, stride, sample=True, check=False)
    xs, vs, xo, vo, fb = oracle.c_rk4_batch2(m, C, x0, v0, dt, nsteps, stride)
    event(f"diverged systems: {'some' if fb.any() else 'none'}; special values: {special}")
    assert res.first_bad.cpu().numpy().tolist() == fb.tolist()
    ok = fb == 0
    gx, gv = res.xs.cpu().numpy(), res.vs.cpu().numpy()
    assert bits(gx[..., ok]) == bits(xs[..., ok]) and bits(gv[..., ok]) == bits(vs[..., ok])
    assert bits(res.x.cpu().numpy()[:, ok]) == bits(xo[:, ok])
    assert bits(res.v.cpu().numpy()[:, ok]) == bits(vo[:, ok])


@SETTINGS
@given(B=st.integers(1, 6), s=st.one_of(st.integers(1, 2048), st.integers(2049, 12_000)), nsteps=st.integers(1, 120),
       sdiv=st.integers(1, 4), halo=st.integers(0, 40), dt=DT, seed=st.integers(0, 2**32 - 1),
       special=st.booleans())
def test_chains_random(B, s, nsteps, sdiv, halo, dt, seed, special):
    rng = np.random.default_rng(seed)
    m, C, x0, v0 = _draw_state(rng, (B, s), special)
    stride = max(1, nsteps // sdiv)
    res = batched.integrate_chains(m, C, x0, v0, dt, nsteps, stride, sample=True, check=False,
                                   halo_steps=halo)
    xs, vs, xo, vo, fb = oracle.c_rk4_chains(m, C, x0, v0, dt, nsteps, stride)
    event(f"{'tiled' if s > 2048 else 'whole-chain'}; diverged: {'some' if fb.any() else 'none'}")
    assert res.first_bad.cpu().numpy().tolist() == fb.tolist()
    ok = fb == 0
    gx, gv = res.xs.cpu().numpy(), res.vs.cpu().numpy()
    assert bits(gx[:, ok]) == bits(xs[:, ok]) and bits(gv[:, ok]) == bits(vs[:, ok])
    assert bits(res.x.cpu().numpy()[ok]) == bits(xo[ok])
