"""Edge cases of the GPU path against the byte-identical oracle: operands that
leave the division fast path (zeros, subnormals, near-overflow, subnormal
masses), sampling edge cases, odd chain lengths around the tile size, and
divergence on the very first step.  Bar: byte-equal, same first bad step."""

import numpy as np
import pytest

import oracle
from conftest import bits

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_1702_02207_b200 import batched  # noqa: E402


def _check_batch2(m, C, x0, v0, dt, nsteps, stride):
    res = batched.integrate_batch2(m, C, x0, v0, dt, nsteps, stride, sample=True, check=False)
    xs, vs, _, _, fb = oracle.c_rk4_batch2(m, C, x0, v0, dt, nsteps, stride)
    got_fb = res.first_bad.cpu().numpy()
    assert got_fb.tolist() == fb.tolist()
    ok = fb == 0
    gx, gv = res.xs.cpu().numpy(), res.vs.cpu().numpy()
    assert bits(gx[..., ok]) == bits(xs[..., ok]) and bits(gv[..., ok]) == bits(vs[..., ok])
    # samples strictly before each diverged system's bad step are exact too
    for b in np.nonzero(~ok)[0]:
        n_ok = 1 + (int(fb[b]) - 1) // stride
        assert bits(gx[:n_ok, :, b]) == bits(xs[:n_ok, :, b])
    return res, fb


def test_slow_path_operands_batch2():
    rng = np.random.default_rng(99)
    B = 4096
    m = rng.uniform(0.5, 2.0, (2, B))
    C = rng.uniform(500.0, 2000.0, (2, B))
    x0 = rng.standard_normal((2, B))
    v0 = rng.standard_normal((2, B))
    x0[:, 0:64] = 0.0                 # equilibrium: zero numerators every step
    v0[:, 0:64] = 0.0
    x0[0, 64:128] = -0.0              # signed zeros
    x0[:, 128:192] = 1e-310           # subnormal positions: tiny numerators
    v0[:, 128:192] = 0.0
    x0[:, 192:256] = 1e-200           # tiny but normal
    x0[:, 256:320] = 1e150            # huge but finite
    m[:, 320:384] = 5e-324            # subnormal masses (valid: positive, finite)
    m[:, 384:448] = 1e300             # huge masses
    C[:, 448:512] = 1e-300            # tiny springs
    _check_batch2(m, C, x0, v0, 1e-4, 500, 100)


def test_two_operation_division_range_edges():
    """Masses at and around the two-operation division's admissible range
    (2^-100 <= m < 2^101) and state magnitudes around its numerator range
    (2^-500 <= |a| < 2^501): inside it the systems run the two-operation
    loop, outside the three-operation one or the exact replay; every system
    byte-equal to the oracle."""
    rng = np.random.default_rng(5)
    edges = np.array([2.0 ** -100, np.nextafter(2.0 ** -100, 0), 2.0 ** 101,
                      np.nextafter(2.0 ** 101, 0), 2.0 ** -100 * 1.5, 2.0 ** 100 * 1.7, 1.0, 0.75])
    B = 2048
    m = rng.choice(edges, (2, B))
    C = rng.uniform(500.0, 2000.0, (2, B)) * m  # keep omega^2 = C/m moderate
    x0 = rng.standard_normal((2, B))
    v0 = np.zeros((2, B))
    scale = rng.choice([1.0, 2.0 ** -490, 2.0 ** -505, 2.0 ** 490, 2.0 ** 505], B)
    x0 *= scale
    cls = batched.div2_classify(m).cpu().numpy()
    assert (cls == 0).any() and (cls != 0).any()
    _check_batch2(m, C, x0, v0, 1e-4, 300, 100)


@pytest.mark.parametrize("shape", ["2,256", "1,128"])
def test_batch2_state_range_edges(shape, monkeypatch):
    """The two-systems-per-thread build tests the range of the step's START
    state instead of every quotient (2^-300 <= |x| < 2^300, |v| < 2^300,
    2^-100 <= C < 2^101; osc_device.cuh, div2s).  Systems on both sides of
    every edge, far outside, exact zeros and subnormals: byte-equal to the
    oracle, through the untested loop, the three-operation loop or the exact
    replay; the one-system build (numerator tests) sees the same inputs."""
    monkeypatch.setenv("OSC_B2", shape)
    rng = np.random.default_rng(41)
    B = 8192
    m = rng.uniform(0.5, 2.0, (2, B))
    C = rng.uniform(500.0, 2000.0, (2, B))
    x0 = rng.standard_normal((2, B))
    v0 = rng.standard_normal((2, B))
    lo, hi = 2.0 ** -300, 2.0 ** 300
    xe = np.array([lo, np.nextafter(lo, 0.0), -lo, 2.0 ** -301, 2.0 ** -353, 2.0 ** -700, 5e-324,
                   0.0, -0.0, np.nextafter(hi, 0.0), hi, -hi, 2.0 ** 305, 2.0 ** 299])
    ve = np.array([np.nextafter(hi, 0.0), hi, -hi, 2.0 ** 310, 0.0, -0.0, 2.0 ** -900, 5e-324])
    Ce = np.array([2.0 ** -100, np.nextafter(2.0 ** -100, 0.0), 2.0 ** -120, 2.0 ** -90, 2.0 ** 18])
    pick = rng.permutation(B)
    k = 0
    for arr, vals in ((x0, xe), (v0, ve), (C, Ce)):
        for val in vals:
            for dof in (0, 1):          # each value in either coordinate, ...
                arr[dof, pick[k]] = val
                k += 1
            arr[:, pick[k]] = val       # ... and in both
            k += 1
    _check_batch2(m, C, x0, v0, 1e-4, 200, 50)


@pytest.mark.parametrize("shape", ["2,256", "1,128"])
def test_batch2_equal_positions_keep_the_sign_of_zero(shape, monkeypatch):
    """x1 == x2 makes the second coordinate's numerator -(C2*(x2 - x1)) = -0,
    and (-0)/m = -0: with very soft springs the two positions stay equal for
    many steps and a velocity that starts at -0.0 must stay -0.0.  A
    two-operation quotient RN(a*zh + RN(a*zl)) of a = -0 is +0 when zl < 0, so
    the untested loop negates the quotient, not the numerator (accel2)."""
    monkeypatch.setenv("OSC_B2", shape)
    rng = np.random.default_rng(7)
    B = 4096
    m = rng.uniform(0.5, 2.0, (2, B))
    C = np.full((2, B), 2.0 ** -90)
    x0 = np.ones((2, B)) * rng.uniform(0.5, 2.0, B)
    v0 = np.full((2, B), -0.0)
    cls = batched.div2_classify(m).cpu().numpy()
    assert (cls != 0).all(axis=0).mean() > 0.9   # the two-operation loop runs
    res, fb = _check_batch2(m, C, x0, v0, 1e-4, 8, 4)
    assert not fb.any()
    v1 = res.vs.cpu().numpy()[-1, 1]
    assert (v1 == 0).all() and np.signbit(v1).all()


@pytest.mark.parametrize("shape", ["2,256", "1,128", "1,32"])
def test_batch2_divergence_in_later_chunks(shape, monkeypatch):
    """Systems just past RK4's stability limit overflow after hundreds to
    thousands of steps: their first bad step falls in the 1st to 8th chunk of
    K1's time loop (512 steps between divergence checks), in chunks whose
    other systems are still fine or have not diverged yet.  First bad step,
    every sample before it and every surviving system: the reference's."""
    monkeypatch.setenv("OSC_B2", shape)
    rng = np.random.default_rng(11)
    B, dt = 256, 1e-3
    m = rng.uniform(0.5, 2.0, (2, B))
    wdt = rng.uniform(2.85, 3.3, B)              # omega*dt around the limit 2.83
    C = (wdt / dt) ** 2 * m / rng.uniform(2.0, 3.0, (2, B))
    x0 = rng.standard_normal((2, B))
    v0 = rng.standard_normal((2, B))
    _, fb = _check_batch2(m, C, x0, v0, dt, 4000, 500)
    late = fb[fb > 0]
    assert (late > 512).sum() > 50 and (late > 1536).sum() > 10 and (fb == 0).sum() > 10


def test_stride_not_dividing_nsteps():
    rng = np.random.default_rng(5)
    m, C = rng.uniform(0.5, 2, (2, 1000)), rng.uniform(500, 2000, (2, 1000))
    x0, v0 = rng.standard_normal((2, 1000)), np.zeros((2, 1000))
    res, _ = _check_batch2(m, C, x0, v0, 1e-4, 1001, 300)
    assert res.xs.shape[0] == 4
    _, _, xf, vf, _ = oracle.c_rk4_batch2(m, C, x0, v0, 1e-4, 1001, sample=False)
    assert bits(res.x.cpu().numpy()) == bits(xf)  # final state is step 1001, not a sample


def test_divergence_on_first_step_and_overflow():
    m = np.array([[1.0, 1.0, 1.0], [1.0, 1.0, 1.0]])
    C = np.array([[1.0, 1e308, 1.0], [1.0, 1e308, 1.0]])
    x0 = np.array([[1.0, 1.0, 1e308], [0.0, -1.0, -1e308]])
    v0 = np.zeros((2, 3))
    _, fb = _check_batch2(m, C, x0, v0, 1.0, 50, 1)
    assert fb[1] == 1 and fb[2] >= 1


@pytest.mark.parametrize("s", [2047, 2048, 2049, 2050, 4095, 4097, 6001])
def test_chain_lengths_around_tile(s):
    """Whole-chain vs tiled, persistent (even) vs plain tiled (odd) lengths."""
    rng = np.random.default_rng(s)
    m = rng.uniform(0.5, 2.0, s)
    C = rng.uniform(500.0, 2000.0, s)
    x0 = rng.standard_normal(s)
    v0 = rng.standard_normal(s)
    res = batched.integrate_chains(m, C, x0, v0, 1e-3, 130, 65, sample=True)
    xs, vs, _, _, fb = oracle.c_rk4_chains(m[None], C[None], x0[None], v0[None], 1e-3, 130, 65)
    assert bits(res.xs.cpu().numpy()) == bits(xs) and bits(res.vs.cpu().numpy()) == bits(vs)


def test_chain_slow_path_cells():
    """Zero / subnormal / signed-zero cells inside a long tiled chain force the
    exact replay of their tiles; the bytes must not change."""
    s = 9000
    rng = np.random.default_rng(17)
    m = rng.uniform(0.5, 2.0, s)
    C = rng.uniform(500.0, 2000.0, s)
    x0 = rng.standard_normal(s)
    v0 = rng.standard_normal(s)
    x0[1000:1500] = 0.0
    v0[1000:1500] = 0.0
    x0[3000:3010] = 1e-310
    x0[5000] = -0.0
    m[7000] = 5e-324
    res = batched.integrate_chains(m, C, x0, v0, 1e-4, 200, check=False)
    _, _, xo, vo, fb = oracle.c_rk4_chains(m[None], C[None], x0[None], v0[None], 1e-4, 200,
                                           sample=False)
    assert int(res.first_bad[0]) == int(fb[0])
    if fb[0] == 0:
        assert bits(res.x.cpu().numpy()) == bits(xo) and bits(res.v.cpu().numpy()) == bits(vo)


@pytest.mark.parametrize("shape", ["tiled", "whole"])
def test_chain_state_range_edges(shape):
    """Chain cells at extreme magnitudes: positions around 2^-300 and 2^300 (and
    far outside: 2^-700, subnormal, exact zeros), velocities up to 2^310 and
    down to subnormal, spring constants at 2^-100, 2^-120 and -- in chains of
    their own, which then diverge -- around 2^101.  Every cell must give the
    reference's bytes (and the diverging chains its first bad step), through
    the two-operation loops or through the exact replay.  (Written for a
    build that range-tested the step's start state instead of each quotient,
    profiles/r02/README.md; the values sit on both sides of its edges.)"""
    rng = np.random.default_rng(31)
    B, s = (1, 12000) if shape == "tiled" else (16, 1024)
    m = rng.uniform(0.5, 2.0, (B, s))
    C = rng.uniform(500.0, 2000.0, (B, s))
    x0 = rng.standard_normal((B, s))
    v0 = rng.standard_normal((B, s))
    lo, hi = 2.0 ** -300, 2.0 ** 300
    xs_edge = [lo, np.nextafter(lo, 0.0), -lo, lo * 1.5, 2.0 ** -301, 2.0 ** -353, 2.0 ** -700,
               np.nextafter(hi, 0.0), hi, -hi, 2.0 ** 299, 2.0 ** 305, 0.0, -0.0, 5e-324]
    vs_edge = [np.nextafter(hi, 0.0), hi, -hi, 2.0 ** 310, 0.0, 2.0 ** -900, 5e-324, -2.0 ** -320]
    Cs_edge = [2.0 ** -100, np.nextafter(2.0 ** -100, 0.0), 2.0 ** -120, 2.0 ** 18]
    # the upper edge of the spring range makes RK4 diverge at any usable dt:
    # those go into chains of their own (whole shape), whose first bad step
    # must be the reference's
    Cs_top = [np.nextafter(2.0 ** 101, 0.0), 2.0 ** 101, 2.0 ** 100] if shape == "whole" else []
    if shape == "tiled":
        # spread over the chain: different tiles, tile edges (2048-cell tiles) included
        cells = rng.choice(np.arange(2, s - 2), size=len(xs_edge) + len(vs_edge) + len(Cs_edge),
                           replace=False)
        where = [(0, int(c)) for c in cells]
    else:
        # one edge value per chain where possible, first / last / interior cells
        n = len(xs_edge) + len(vs_edge) + len(Cs_edge)
        where = [(i % (B - 3), int(c)) for i, c in enumerate(rng.choice(np.arange(s), size=n,
                                                                        replace=False))]
    it = iter(where)
    for val in xs_edge:
        b, c = next(it)
        x0[b, c] = val
    for val in vs_edge:
        b, c = next(it)
        v0[b, c] = val
    for val in Cs_edge:
        b, c = next(it)
        C[b, c] = val
    for i, val in enumerate(Cs_top):
        C[B - 1 - i, 100 + 300 * i] = val
    args = (m[0], C[0], x0[0], v0[0]) if B == 1 else (m, C, x0, v0)
    res = batched.integrate_chains(*args, 1e-4, 90, check=False)
    _, _, xo, vo, fb = oracle.c_rk4_chains(m, C, x0, v0, 1e-4, 90, sample=False)
    assert res.first_bad.cpu().numpy().reshape(-1).tolist() == fb.tolist()
    good = fb == 0
    assert good[: B - len(Cs_top)].all() and not good[B - len(Cs_top):].any()
    assert bits(res.x.cpu().numpy().reshape(B, s)[good]) == bits(xo[good])
    assert bits(res.v.cpu().numpy().reshape(B, s)[good]) == bits(vo[good])


def test_many_small_chains_whole_chain_mode():
    """B chains of odd small lengths (padded CTAs)."""
    for s in (3, 17, 100, 513):
        rng = np.random.default_rng(s)
        B = 37
        m = rng.uniform(0.5, 2.0, (B, s))
        C = rng.uniform(500.0, 2000.0, (B, s))
        x0 = rng.standard_normal((B, s))
        v0 = rng.standard_normal((B, s))
        x0[5] = 0.0
        v0[5] = 0.0
        res = batched.integrate_chains(m, C, x0, v0, 1e-3, 600)
        _, _, xo, vo, _ = oracle.c_rk4_chains(m, C, x0, v0, 1e-3, 600, sample=False)
        assert bits(res.x.cpu().numpy()) == bits(xo) and bits(res.v.cpu().numpy()) == bits(vo)


def test_batch_parameter_validation_mirrors_reference():
    """OscillatorSystem's rule (oscillator.py:75-80) applied to whole batches."""
    import paper_1702_02207_b200 as osc

    ok = np.ones((2, 4))
    for bad in (0.0, -1.0, np.nan, np.inf):
        m = ok.copy()
        m[1, 2] = bad
        with pytest.raises(osc.NonPositiveParameterError):
            batched.integrate_batch2(m, ok, ok, ok, 1e-3, 5)
        with pytest.raises(osc.NonPositiveParameterError):
            batched.integrate_chains(ok, m, ok, ok, 1e-3, 5)
    # subnormal masses are positive and finite: accepted, as by the reference
    m = ok.copy()
    m[0, 0] = 5e-324
    batched.integrate_batch2(m, ok, ok * 0, ok * 0, 1e-3, 5)


def test_divergence_step_not_lost_to_tile_order():
    """Regression: a tile must not skip because ANOTHER tile of the same
    launch already recorded a (later) divergence step.  Persistent tiled
    kernel, 148 CTAs striding over 170 tiles: tiles 10 and 20 diverge in
    round one (steps ~35, ~36; their exact replays delay their CTAs), tile
    168 -- CTA 20's second tile -- holds the earliest step (~34)."""
    W = 2048 - 4 * 32  # owned cells per tile at the default 32 steps per launch
    s = 170 * W
    rng = np.random.default_rng(21)
    m = rng.uniform(0.5, 2.0, s)
    C = rng.uniform(500.0, 2000.0, s)
    x0 = rng.standard_normal(s)
    v0 = np.zeros(s)
    for tile, c in ((10, 6.0e10), (20, 4.0e10), (168, 9.0e10)):
        C[tile * W + W // 2] = c
    res = batched.integrate_chains(m, C, x0, v0, 1e-3, 64, check=False, halo_steps=32)
    _, _, _, _, fb = oracle.c_rk4_chains(m[None], C[None], x0[None], v0[None], 1e-3, 64,
                                         sample=False)
    assert 32 < fb[0] <= 64
    assert int(res.first_bad[0]) == int(fb[0])


def test_whole_chain_batch_split_over_two_streams():
    """>= 1024 whole chains run as two halves on two streams: samples,
    energies, final states and per-chain divergence steps (one diverging
    chain in each half) equal the oracle's."""
    B, s = 1500, 64
    rng = np.random.default_rng(33)
    m = rng.uniform(0.5, 2.0, (B, s))
    C = rng.uniform(500.0, 2000.0, (B, s))
    x0 = rng.standard_normal((B, s))
    v0 = rng.standard_normal((B, s))
    C[100, 30] = 3e8   # first half diverges
    C[1400, 5] = 5e8   # second half diverges
    res = batched.integrate_chains(m, C, x0, v0, 1e-3, 600, 150, sample=True, energies=True,
                                   check=False)
    xs, vs, xo, vo, fb = oracle.c_rk4_chains(m, C, x0, v0, 1e-3, 600, 150)
    assert res.first_bad.cpu().numpy().tolist() == fb.tolist()
    assert fb[100] > 0 and fb[1400] > 0
    ok = fb == 0
    assert bits(res.xs.cpu().numpy()[:, ok]) == bits(xs[:, ok])
    assert bits(res.x.cpu().numpy()[ok]) == bits(xo[ok])
    es = res.energies.cpu().numpy()
    for k in range(xs.shape[0]):
        assert bits(es[k][ok]) == bits(oracle.c_energy(m[ok], C[ok], xs[k][ok], vs[k][ok]))
