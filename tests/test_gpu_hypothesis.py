"""Property-based parity of the GPU path against the C oracle (which is
pinned to the reference in tests/test_oracle.py): random batches and chains,
random step counts, strides, tile depths and step sizes (stable and
diverging), with +-0, subnormal, tiny and huge entries.  Bar: byte-equal
samples and final states, equal first divergence steps."""

import numpy as np
import pytest
import os as _os
from hypothesis import HealthCheck, event, given, settings, strategies as st

_SOAK = int(_os.environ.get("HYPOTHESIS_SOAK", "1"))  # bug-hunt scaling (scripts/)
# the default run replays a fixed example set (reproducible suite); a soak
# (scripts/hypothesis_soak.sh) explores fresh random examples
_DERANDOMIZE = _SOAK == 1

import oracle
from conftest import bits

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_1702_02207_b200 import batched  # noqa: E402

SETTINGS = settings(max_examples=200 * _SOAK, deadline=None, derandomize=_DERANDOMIZE,
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
            a[k] = rng.choice(_SPECIAL, k.size) * rng.choice([1.0, -1.0], k.size)
    return m, C, x0, v0


# zeros, subnormals, far-out magnitudes, and both sides of the bounds of K1's
# state-range tests (2^-300 <= |x| < 2^300, |v| < 2^300; osc_device.cuh)
_SPECIAL = np.array([0.0, -0.0, 5e-324, 1e-310, 1e-200, 1e150, 2.0 ** -300,
                     np.nextafter(2.0 ** -300, 0.0), 2.0 ** -301, 2.0 ** -299, 2.0 ** 300,
                     np.nextafter(2.0 ** 300, 0.0), 2.0 ** 299, 2.0 ** 301])


def _twin_systems(rng, m, C, x0, v0):
    """A few 2-DOF systems with x1 == x2, zero velocities of either sign and
    very soft springs: the positions stay equal for many steps, the second
    coordinate's numerator is -0 at every stage, and the sign of the zero
    quotient must be the reference's (k_batch2.cu, accel2)."""
    B = m.shape[1]
    k = rng.integers(0, B, max(1, B // 16))
    x0[1, k] = x0[0, k]
    v0[:, k] = rng.choice([0.0, -0.0], (2, k.size))
    C[:, k] = 2.0 ** rng.integers(-99, -60, (2, k.size)).astype(float)


@SETTINGS
@given(B=st.integers(1, 3000), nsteps=st.integers(1, 300), sdiv=st.integers(1, 8),
       dt=DT, seed=st.integers(0, 2**32 - 1), special=st.booleans(), twins=st.booleans())
def test_batch2_random(B, nsteps, sdiv, dt, seed, special, twins):
    rng = np.random.default_rng(seed)
    m, C, x0, v0 = _draw_state(rng, (2, B), special)
    if twins:
        _twin_systems(rng, m, C, x0, v0)
    stride = max(1, nsteps // sdiv + (seed % 3))
    res = batched.integrate_batch2(m, C, x0, v0, dt, nsteps, stride, sample=True, check=False)
    xs, vs, xo, vo, fb = oracle.c_rk4_batch2(m, C, x0, v0, dt, nsteps, stride)
    event(f"diverged systems: {'some' if fb.any() else 'none'}; special values: {special}; "
          f"twin systems: {twins}")
    assert res.first_bad.cpu().numpy().tolist() == fb.tolist()
    ok = fb == 0
    gx, gv = res.xs.cpu().numpy(), res.vs.cpu().numpy()
    assert bits(gx[..., ok]) == bits(xs[..., ok]) and bits(gv[..., ok]) == bits(vs[..., ok])
    assert bits(res.x.cpu().numpy()[:, ok]) == bits(xo[:, ok])
    assert bits(res.v.cpu().numpy()[:, ok]) == bits(vo[:, ok])


_TESTED = []


def _tested_divisors():
    """Masses whose two-operation quotients the chain kernels must test
    (no div2 class: ~0.05% of random masses), drawn once from the device
    table (osc_div2c_table)."""
    if not _TESTED:
        pool = np.random.default_rng(5).uniform(0.5, 2.0, 400_000)
        bad = batched.div2c_table(pool)[2].cpu().numpy().view(np.uint64)
        _TESTED.append(pool[(bad >> np.uint64(63)) == 0])
    return _TESTED[0]


def _inject_divisors(rng, m, kind):
    """kind "tested": ~1% of the masses become tested divisors (scaled by a
    power of two: the class depends on the significand only), so most warps
    run the tested two-operation loop; "ineligible": a few masses outside
    [2^-100, 2^101) send their tiles to the exact replay."""
    flat = m.reshape(-1)
    if kind == "tested":
        k = rng.integers(0, flat.size, max(1, flat.size // 100))
        flat[k] = rng.choice(_tested_divisors(), k.size) * 2.0 ** rng.integers(-3, 4, k.size)
    elif kind == "ineligible":
        k = rng.integers(0, flat.size, max(1, flat.size // 3000))
        flat[k] = 2.0 ** 101 * rng.uniform(1.0, 4.0, k.size)


@SETTINGS
@given(B=st.integers(1, 6), s=st.one_of(st.integers(1, 2048), st.integers(2049, 12_000)), nsteps=st.integers(1, 120),
       sdiv=st.integers(1, 4), halo=st.integers(0, 40), dt=DT, seed=st.integers(0, 2**32 - 1),
       special=st.booleans(), divisors=st.sampled_from(["random", "random", "tested", "ineligible"]))
def test_chains_random(B, s, nsteps, sdiv, halo, dt, seed, special, divisors):
    rng = np.random.default_rng(seed)
    m, C, x0, v0 = _draw_state(rng, (B, s), special)
    _inject_divisors(rng, m, divisors)
    stride = max(1, nsteps // sdiv)
    res = batched.integrate_chains(m, C, x0, v0, dt, nsteps, stride, sample=True, check=False,
                                   halo_steps=halo)
    xs, vs, xo, vo, fb = oracle.c_rk4_chains(m, C, x0, v0, dt, nsteps, stride)
    event(f"{'tiled' if s > 2048 else 'whole-chain'}; divisors: {divisors}; "
          f"diverged: {'some' if fb.any() else 'none'}")
    assert res.first_bad.cpu().numpy().tolist() == fb.tolist()
    ok = fb == 0
    gx, gv = res.xs.cpu().numpy(), res.vs.cpu().numpy()
    assert bits(gx[:, ok]) == bits(xs[:, ok]) and bits(gv[:, ok]) == bits(vs[:, ok])
    assert bits(res.x.cpu().numpy()[ok]) == bits(xo[ok])


@settings(max_examples=30 * _SOAK, deadline=None, derandomize=_DERANDOMIZE, suppress_health_check=[HealthCheck.too_slow])
@given(B=st.integers(1, 700_000), nsteps=st.integers(1, 60), seed=st.integers(0, 2**32 - 1))
def test_batch2_host_path_random(B, nsteps, seed):
    """Host-pointer C ABI (chunked, multi-stream) == device path, bit for bit."""
    from paper_1702_02207_b200 import _native

    rng = np.random.default_rng(seed)
    m, C, x0, v0 = _draw_state(rng, (2, B), seed % 2 == 0)
    x, v = x0.copy(), v0.copy()
    fb = np.zeros(B, dtype=np.int64)
    rc = _native.lib().osc_rk4_batch2_host(m.ctypes.data, C.ctypes.data, x.ctypes.data,
                                           v.ctypes.data, B, 1e-3, nsteps, nsteps, None, None,
                                           fb.ctypes.data)
    res = batched.integrate_batch2(m, C, x0, v0, 1e-3, nsteps, check=False)
    dfb = res.first_bad.cpu().numpy()
    assert fb.tolist() == dfb.tolist()
    assert rc == (_native.OSC_NONFINITE if dfb.any() else _native.OSC_OK)
    ok = dfb == 0
    assert bits(x[:, ok]) == bits(res.x.cpu().numpy()[:, ok])
    assert bits(v[:, ok]) == bits(res.v.cpu().numpy()[:, ok])


@settings(max_examples=40 * _SOAK, deadline=None, derandomize=_DERANDOMIZE, suppress_health_check=[HealthCheck.too_slow])
@given(B=st.integers(1, 500), nsteps=st.integers(1, 80), sdiv=st.integers(1, 5),
       seed=st.integers(0, 2**32 - 1), chains=st.booleans(), s=st.integers(1, 3000))
def test_sample_energies_random(B, nsteps, sdiv, seed, chains, s):
    """energy() of every retained sample, computed on the device, equals the
    (reference-pinned) oracle's energy of the same sample bit for bit."""
    rng = np.random.default_rng(seed)
    stride = max(1, nsteps // sdiv)
    if chains:
        B = min(B, 4)
        m, C, x0, v0 = _draw_state(rng, (B, s), False)
        res = batched.integrate_chains(m, C, x0, v0, 1e-4, nsteps, stride, sample=True,
                                       energies=True, check=False)
        xs, vs = res.xs.cpu().numpy(), res.vs.cpu().numpy()  # [nsamp][B][s]
        es = res.energies.cpu().numpy()
        for k in range(xs.shape[0]):
            assert bits(es[k]) == bits(oracle.c_energy(m, C, xs[k], vs[k]))
    else:
        m, C, x0, v0 = _draw_state(rng, (2, B), False)
        res = batched.integrate_batch2(m, C, x0, v0, 1e-4, nsteps, stride, sample=True,
                                       energies=True, check=False)
        xs, vs = res.xs.cpu().numpy(), res.vs.cpu().numpy()  # [nsamp][2][B]
        es = res.energies.cpu().numpy()
        for k in range(xs.shape[0]):
            assert bits(es[k]) == bits(oracle.c_energy(m.T, C.T, xs[k].T, vs[k].T))


@settings(max_examples=25 * _SOAK, deadline=None, derandomize=_DERANDOMIZE, suppress_health_check=[HealthCheck.too_slow])
@given(s=st.integers(1, 300), N=st.integers(1, 90), nsteps=st.integers(1, 25),
       seed=st.integers(0, 2**32 - 1))
def test_dense_random_shapes(s, N, nsteps, seed):
    """Padded dense path (s -> x128, N -> x32) vs the numpy restatement,
    relative 1e-10 (GEMM summation order)."""
    rng = np.random.default_rng(seed)
    m = rng.uniform(0.5, 2.0, s)
    q, _ = np.linalg.qr(rng.standard_normal((s, s)))
    K = (q * rng.uniform(500.0, 2000.0, s)) @ q.T
    K = 0.5 * (K + K.T)
    A = K / m[:, None]
    X0, V0 = rng.standard_normal((s, N)), rng.standard_normal((s, N))
    res = batched.integrate_dense(A, X0, V0, 1e-4, nsteps)
    Xo, Vo = oracle.dense_rk4(A, X0, V0, 1e-4, nsteps)
    for got, ref in ((res.x.cpu().numpy(), Xo), (res.v.cpu().numpy(), Vo)):
        assert np.max(np.abs(got - ref)) <= 1e-10 * max(1.0, np.max(np.abs(ref)))


@settings(max_examples=60 * _SOAK, deadline=None, derandomize=_DERANDOMIZE,
          suppress_health_check=[HealthCheck.too_slow])
@given(B=st.integers(1, 64), s=st.integers(1, 600), seed=st.integers(0, 2**32 - 1),
       special=st.booleans(), cell_major=st.booleans())
def test_host_derivative_energy_random(B, s, seed, special, cell_major):
    """The staged one-round-trip host forms (osc_derivative_host /
    osc_energy_host, parameter rule fused into the kernels) equal the oracle
    bit for bit, in both layouts."""
    import ctypes

    from paper_1702_02207_b200 import _native

    lib = _native.lib()
    rng = np.random.default_rng(seed)
    m, C, x0, v0 = _draw_state(rng, (B, s), special)
    dref = oracle.c_derivative(m, C, x0)
    eref = oracle.c_energy(m, C, x0, v0)
    if cell_major:  # [s][B]
        m, C, x0, v0 = (np.ascontiguousarray(a.T) for a in (m, C, x0, v0))
    dv = np.empty_like(x0)
    e = np.empty(B)
    p = lambda a: ctypes.c_void_p(a.ctypes.data)  # noqa: E731
    assert lib.osc_derivative_host(p(m), p(C), p(x0), p(dv), B, s, int(cell_major)) == 0
    assert lib.osc_energy_host(p(m), p(C), p(x0), p(v0), p(e), B, s, int(cell_major)) == 0
    got = dv.T if cell_major else dv
    with np.errstate(all="ignore"):
        assert bits(np.nan_to_num(got, nan=7.0)) == bits(np.nan_to_num(dref, nan=7.0))
        assert bits(np.nan_to_num(e, nan=7.0)) == bits(np.nan_to_num(eref, nan=7.0))
