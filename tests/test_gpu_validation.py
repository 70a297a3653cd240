"""The parameter rule at the C ABI (OscillatorSystem, oscillator.py:66-80):
every entry point that takes masses and spring rates rejects a non-finite or
non-positive one with OSC_INVALID before integrating, names the first
offender (masses before springs, lowest index -- the reference's order), and
leaves the caller's host outputs untouched.  Plus the bulk-copy alignment
rule of the persistent tile kernel (misaligned views fall back, same bytes).
"""

import ctypes

import numpy as np
import pytest

import oracle
from conftest import bits

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_1702_02207_b200 import _native, batched, workloads  # noqa: E402
from paper_1702_02207_b200 import oscillator as osc  # noqa: E402

BAD = [float("nan"), float("inf"), float("-inf"), -1.0, 0.0, -0.0, -5e-324]

lib = _native.lib()
P = ctypes.c_void_p


def _p(t):
    return P(t.data_ptr()) if isinstance(t, torch.Tensor) else P(t.ctypes.data)


def _last():
    return _native.last_invalid_parameter()


def _stream():
    return P(torch.cuda.current_stream().cuda_stream)


@pytest.mark.parametrize("bad", BAD)
@pytest.mark.parametrize("which", [0, 1])
def test_batch2_device_entry_rejects(bad, which):
    m, C, x0, v0 = (torch.from_numpy(a).cuda() for a in workloads.c2(B=1000))
    arrs = [m, C]
    arrs[which][1, 17] = bad  # coordinate 1 of system 17: flat index B + 17
    fb = torch.zeros(1000, dtype=torch.int64, device="cuda")
    x, v = x0.clone(), v0.clone()
    rc = lib.osc_rk4_batch2(_p(m), _p(C), _p(x), _p(v), 1000, 1e-4, 50, 50, None, None, None,
                            _p(fb), 0, _stream())
    assert rc == _native.OSC_INVALID
    assert _last() == (which, 1017)
    msg = _native.last_error()
    assert msg.startswith(("masses[1]", "springs[1]")[which]) and "(system 17)" in msg
    torch.cuda.synchronize()
    assert torch.equal(x, x0)  # nothing was enqueued
    with pytest.raises(osc.NonPositiveParameterError, match=r"\[1, 17\]"):
        batched.integrate_batch2(m, C, x0, v0, 1e-4, 50)
    # OSC_TRUSTED: the caller vouches for the parameters; no check
    rc = lib.osc_rk4_batch2(_p(m), _p(C), _p(x), _p(v), 1000, 1e-4, 50, 50, None, None, None,
                            _p(fb), _native.OSC_TRUSTED, _stream())
    assert rc == _native.OSC_OK  # (the record, like errno, is kept until the next error)


def test_masses_are_reported_before_springs():
    m, C, x0, v0 = workloads.c4(B=3, s=100)
    C[0, 0] = -1.0  # an earlier spring ...
    m[2, 99] = 0.0  # ... but a mass is bad: the reference checks masses first
    md, Cd, xd, vd = (torch.from_numpy(a).cuda() for a in (m, C, x0, v0))
    with pytest.raises(osc.NonPositiveParameterError, match=r"masses\[2, 99\] = 0\.0"):
        batched.integrate_chains(md, Cd, xd, vd, 1e-4, 10)
    assert _last() == (0, 299)
    m[2, 99] = 1.0
    with pytest.raises(osc.NonPositiveParameterError, match=r"springs\[0, 0\] = -1\.0"):
        batched.integrate_chains(m, C, x0, v0, 1e-4, 10)
    assert "(chain 0)" in _native.last_error()


@pytest.mark.parametrize("s", [2, 7, 5000])
def test_host_forms_reject_and_leave_outputs_untouched(s):
    B = 4
    if s == 2:
        m, C, x0, v0 = workloads.c2(B=B)
    else:
        m, C, x0, v0 = workloads.c4(B=B, s=s)
    m = m.copy()
    m.flat[m.size - 1] = float("nan")
    x, v = x0.copy(), v0.copy()
    xs = np.full((3,) + x.shape, 7.0)
    vs = np.full((3,) + x.shape, 7.0)
    fb = np.full(B, -3, dtype=np.int64)
    if s == 2:
        rc = lib.osc_rk4_batch2_host(_p(m), _p(C), _p(x), _p(v), B, 1e-4, 20, 10, _p(xs),
                                     _p(vs), _p(fb))
    else:
        rc = lib.osc_rk4_chains_host(_p(m), _p(C), _p(x), _p(v), B, s, 1e-4, 20, 10, _p(xs),
                                     _p(vs), _p(fb))
    assert rc == _native.OSC_INVALID
    assert _last() == (0, m.size - 1)
    assert bits(x) == bits(x0) and bits(v) == bits(v0)
    assert (xs == 7.0).all() and (vs == 7.0).all() and (fb == -3).all()


def test_large_host_run_rejects_before_touching_outputs():
    """The chunked pipeline (> 8 MB) checks every chunk's parameters first."""
    m, C, x0, v0 = workloads.c2(B=1 << 20)
    C = C.copy()
    C[0, 700_001] = float("inf")
    x, v = x0.copy(), v0.copy()
    fb = np.zeros(1 << 20, dtype=np.int64)
    rc = lib.osc_rk4_batch2_host(_p(m), _p(C), _p(x), _p(v), 1 << 20, 1e-4, 10, 10, None, None,
                                 _p(fb))
    assert rc == _native.OSC_INVALID and _last() == (1, 700_001)
    assert bits(x) == bits(x0)


def test_other_entry_points_reject():
    m, C, x0, v0 = workloads.c4(B=1, s=40)
    m = m[0].copy()
    C, x0, v0 = C[0], x0[0], v0[0]
    m[3] = -2.0
    md, Cd, xd, vd = (torch.from_numpy(a).cuda() for a in (m, C, x0, v0))
    s = 40
    out = torch.empty(s, dtype=torch.float64, device="cuda")
    fb = torch.zeros(1, dtype=torch.int64, device="cuda")
    ns = torch.zeros(10, dtype=torch.int64, device="cuda")
    st = _stream()
    calls = {
        "osc_derivative": lambda: lib.osc_derivative(_p(md), _p(Cd), _p(xd), _p(out), 1, s, 0, st),
        "osc_energy": lambda: lib.osc_energy(_p(md), _p(Cd), _p(xd), _p(vd), _p(out), 1, s, 0, st),
        "osc_equation_engine": lambda: lib.osc_equation_engine(
            _p(md), _p(Cd), _p(xd), _p(vd), s, 1e-4, 10, 10, None, None, _p(fb), _p(ns), st),
        "osc_rk4_chain_advance": lambda: lib.osc_rk4_chain_advance(
            _p(md), _p(Cd), _p(xd), _p(vd), _p(out), _p(out), s, 0, s, 1e-4, 4, 0, _p(fb), None,
            None, None, 0, st),
        "osc_rk4_chains": lambda: lib.osc_rk4_chains(
            _p(md), _p(Cd), _p(xd.clone()), _p(vd.clone()), 1, s, 1e-4, 10, 10, None, None, None,
            _p(fb), 0, 0, st),
        "osc_validate_parameters": lambda: lib.osc_validate_parameters(
            _p(md), _p(Cd), s, None, st),
    }
    for name, call in calls.items():
        assert call() == _native.OSC_INVALID, name
        assert _last() == (0, 3), name
    # host forms and the single-process sharded chain
    dv = np.empty(s)
    assert lib.osc_derivative_host(_p(m), _p(C), _p(x0), _p(dv), 1, s, 0) == _native.OSC_INVALID
    assert lib.osc_energy_host(_p(m), _p(C), _p(x0), _p(v0), _p(dv), 1, s, 0) == \
        _native.OSC_INVALID
    devs = (ctypes.c_int * 2)(0, 0)
    m2, C2, x2, v2 = workloads.c3(s=9000)
    C2 = C2.copy()
    C2[8000] = 0.0
    x2c = x2.copy()
    fbh = np.zeros(1, dtype=np.int64)
    rc = lib.osc_rk4_chain_sharded(2, devs, _p(m2), _p(C2), _p(x2), _p(v2), 9000, 1e-4, 10, 0,
                                   _p(fbh), 0)
    assert rc == _native.OSC_INVALID and _last() == (1, 8000)
    assert bits(x2) == bits(x2c)
    # rowscale divides by the masses only
    K = torch.eye(s, dtype=torch.float64, device="cuda")
    with pytest.raises(osc.NonPositiveParameterError, match=r"masses\[3\] = -2\.0"):
        batched.rowscale(K, md)
    bad = ctypes.c_int64(0)
    assert lib.osc_validate_parameters(_p(md), _p(Cd), s, ctypes.byref(bad), st) == \
        _native.OSC_INVALID and bad.value == 3
    # a non-parameter error clears the record
    assert lib.osc_rk4_chains(None, None, None, None, 1, 4, -1.0, 1, 1, None, None, None, None, 0,
                              0, None) == _native.OSC_INVALID
    assert _last() is None


def test_valid_parameters_pass_and_match_oracle():
    m, C, x0, v0 = workloads.c4(B=2, s=300)
    res = batched.integrate_chains(m, C, x0, v0, 1e-4, 64)
    _, _, xo, vo, _ = oracle.c_rk4_chains(m, C, x0, v0, 1e-4, 64, sample=False)
    assert bits(res.x.cpu().numpy()) == bits(xo)
    good = lib.osc_validate_parameters(_p(res.x), _p(res.x), 0, None, _stream())
    assert good == _native.OSC_OK


def test_drop_in_rejects_reference_shaped_bad_systems():
    """A duck-typed system that skipped OscillatorSystem's validation is
    still rejected by the ABI (NonPositiveParameterError, the reference's
    type for the rule)."""
    class Sys:
        masses = (1.0, -1.0, 1.0)
        springs = (1.0, 1.0, 1.0)

    state = osc.PhaseState((1.0, 0.0, 0.0), (0.0, 0.0, 0.0))
    with pytest.raises(osc.NonPositiveParameterError, match=r"masses\[1\] = -1\.0"):
        osc.integrate(Sys(), state, 1e-3, 10)
    with pytest.raises(osc.NonPositiveParameterError):
        osc.derivative(Sys(), state)
    with pytest.raises(osc.NonPositiveParameterError):
        osc.energy(Sys(), state)


@pytest.mark.parametrize("offset", [1, 3])
def test_misaligned_views_take_the_plain_tiled_kernel(offset):
    """the persistent kernel's bulk copies need 16-byte aligned
    bases; an 8-byte aligned view (odd storage offset) must not fault and
    must give the same bytes as an aligned copy."""
    s, n = 6000, 70
    m, C, x0, v0 = workloads.c4(B=1, s=s)
    big = [torch.zeros(s + 4, dtype=torch.float64, device="cuda") for _ in range(4)]
    views = []
    for buf, a in zip(big, (m, C, x0, v0)):
        view = buf[offset:offset + s]
        view.copy_(torch.from_numpy(a[0]))
        views.append(view)
    assert views[0].data_ptr() % 16 == 8
    res = batched.integrate_chains(*(t[None] for t in views), 1e-4, n)
    ref = batched.integrate_chains(m, C, x0, v0, 1e-4, n)
    torch.cuda.synchronize()
    assert bits(res.x.cpu().numpy()) == bits(ref.x.cpu().numpy())
    _, _, xo, _, _ = oracle.c_rk4_chains(m, C, x0, v0, 1e-4, n, sample=False)
    assert bits(ref.x.cpu().numpy()) == bits(xo)
    # the raw advance on misaligned in/out buffers (own range even, n even)
    fb = torch.zeros(1, dtype=torch.int64, device="cuda")
    xo_buf = torch.zeros(s + 4, dtype=torch.float64, device="cuda")
    vo_buf = torch.zeros_like(xo_buf)
    batched.chain_advance(views[0], views[1], views[2], views[3], xo_buf[offset:offset + s],
                          vo_buf[offset:offset + s], 0, s, 1e-4, 8, 0, fb)
    ref8 = batched.integrate_chains(m, C, x0, v0, 1e-4, 8)
    torch.cuda.synchronize()
    assert bits(xo_buf[offset:offset + s].cpu().numpy()) == bits(ref8.x[0].cpu().numpy())
