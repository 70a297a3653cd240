"""Array API over the C ABI: batches of systems and chains resident in HBM.

Inputs may be numpy arrays (copied to the current CUDA device) or float64
CUDA tensors (used in place when contiguous).  Work is enqueued on the current
torch stream; results are device tensors.  These are the calls the bench and
the multi-GPU driver make; ``oscillator.integrate`` is the drop-in wrapper.

    integrate_batch2   BASELINE configs 0-1  (K1 batch2_rk4; compare=True fuses
                       modal.compare against the analytic solution)
    analytic_batch2    modal.analytic_solution per system
    compare_batch2     modal.compare over retained samples
    integrate_chains   BASELINE configs 2-3  (K2 whole-chain / K3 tiled)
    chain_advance      one temporally blocked launch over a shard (K3)
"""

from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np
import torch

from . import _native
from .oscillator import NonFiniteStateError, NonPositiveParameterError, accumulated_times


def _stream(stream=None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def _dev(a, device=None) -> torch.Tensor:
    """Contiguous float64 CUDA tensor (no copy when already one).  Work runs
    on the current CUDA device (the stream is its current stream), so a
    tensor on another GPU is refused rather than launched against."""
    if isinstance(a, torch.Tensor):
        t = a
        if not t.is_cuda:
            t = t.to(device or torch.device("cuda", torch.cuda.current_device()))
        elif t.device.index != torch.cuda.current_device():
            raise ValueError(f"tensor on {t.device} but the current device is "
                             f"cuda:{torch.cuda.current_device()}; call inside "
                             f"torch.cuda.device({t.device})")
    else:
        t = torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).to(
            device or torch.device("cuda", torch.cuda.current_device()))
    if t.dtype != torch.float64:
        raise TypeError(f"expected float64, got {t.dtype}")
    return t.contiguous()


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else None


def raise_for(rc: int, what: str, params=None):
    """Map an OSC_* status to the reference's exception types.  A violated
    parameter rule (the ABI's own check, osc_last_invalid_parameter) becomes
    NonPositiveParameterError naming the element of ``params = (m, C)``."""
    if rc == _native.OSC_OK:
        return
    msg = f"{what}: {_native.last_error()}"
    if rc == _native.OSC_INVALID:
        bad = _native.last_invalid_parameter()
        if bad is not None:
            which, index = bad
            label = ("masses", "springs")[which]
            if params is not None:
                arr = params[which]
                idx = tuple(int(i) for i in np.unravel_index(index, tuple(arr.shape)))
                value = float(arr[idx])
                raise NonPositiveParameterError(
                    f"{label}{list(idx)} = {value!r}; must be positive and finite")
            raise NonPositiveParameterError(msg)
        raise ValueError(msg)
    if rc == _native.OSC_NONFINITE:
        raise NonFiniteStateError(msg)
    raise RuntimeError(msg)


@dataclass
class BatchResult:
    """Final state, optional samples and per-system first bad step (device)."""

    x: torch.Tensor
    v: torch.Tensor
    xs: torch.Tensor | None
    vs: torch.Tensor | None
    first_bad: torch.Tensor
    dt: float
    nsteps: int
    stride: int
    t0: float = 0.0
    energies: torch.Tensor | None = None  # [nsamp][B] energy() of each sample
    errors: "ErrorReports | None" = None  # compare() vs the analytic solution

    def energy_drift(self) -> torch.Tensor:
        """max_k |E_k - E_0| / E_0 per system (harness.py:508-510's drift)."""
        if self.energies is None:
            raise ValueError("run with energies=True")
        e0 = self.energies[0]
        d = (self.energies - e0).abs().amax(dim=0)
        return torch.where(e0 > 0, d / e0, d)

    def times(self) -> np.ndarray:
        return accumulated_times(self.t0, self.dt, self.nsteps, self.stride)

    def check(self):
        """Raise NonFiniteStateError(step=earliest) if any system diverged."""
        if self.first_bad.numel() == 0:
            return self
        fb = self.first_bad
        nz = fb[fb > 0]
        if nz.numel():
            step = int(nz.min().item())
            idx = int(torch.nonzero(fb == step)[0, 0].item())
            raise NonFiniteStateError(
                f"integration diverged at step {step} (system {idx})", step=step)
        return self


@dataclass
class ErrorReports:
    """modal.ErrorReport (modal.py:65-71) for every system of a batch, [B]
    each; NaN for a system that diverged (integrate would have raised)."""

    max_abs_error: torch.Tensor
    rmse: torch.Tensor
    at_time: torch.Tensor


MODAL_FIELDS = ("omega1", "omega2", "r1", "r2", "a1c", "a1s", "a2c", "a2s")


def analytic_batch2(m, C, x0, v0, *, stream=None) -> torch.Tensor:
    """modal.analytic_solution (modal.py:98-120) per system, ``[8][B]`` in
    MODAL_FIELDS order.  Equal parameters give the reference's bits; unequal
    ones the general two-mode solution of the 2x2 pencil (osc_modal.cuh)."""
    lib = _native.lib()
    m, C, x0, v0 = (_dev(a) for a in (m, C, x0, v0))
    if m.dim() != 2 or m.shape[0] != 2 or not (m.shape == C.shape == x0.shape == v0.shape):
        raise ValueError(f"expected [2][B] arrays, got {tuple(m.shape)}")
    B = m.shape[1]
    sol = torch.empty((len(MODAL_FIELDS), B), dtype=torch.float64, device=m.device)
    rc = lib.osc_analytic_batch2(_ptr(m), _ptr(C), _ptr(x0), _ptr(v0), B, _ptr(sol),
                                 ctypes.c_void_p(_stream(stream)))
    raise_for(rc, "osc_analytic_batch2", (m, C))
    return sol


def _reports(out: torch.Tensor) -> ErrorReports:
    return ErrorReports(out[0], out[1], out[2])


def compare_batch2(sol, xs, ts, *, stream=None) -> ErrorReports:
    """modal.compare (modal.py:141-162) of retained samples ``xs``
    ``[nsamp][2][B]`` at time labels ``ts`` against ``sol`` ``[8][B]``."""
    lib = _native.lib()
    sol, xs, ts = _dev(sol), _dev(xs), _dev(ts)
    if xs.dim() != 3 or xs.shape[1] != 2 or ts.shape != (xs.shape[0],):
        raise ValueError("expected xs [nsamp][2][B] and ts [nsamp]")
    B = xs.shape[2]
    if sol.shape != (len(MODAL_FIELDS), B):
        raise ValueError(f"expected sol [8][{B}], got {tuple(sol.shape)}")
    out = torch.empty((3, B), dtype=torch.float64, device=xs.device)
    rc = lib.osc_compare_batch2(_ptr(sol), _ptr(xs), _ptr(ts), xs.shape[0], B, _ptr(out),
                                ctypes.c_void_p(_stream(stream)))
    raise_for(rc, "osc_compare_batch2")
    return _reports(out)


def _outputs(x0, v0, nsteps, stride, sample):
    x = x0.clone()
    v = v0.clone()
    xs = vs = None
    if sample:
        nsamp = 1 + nsteps // stride
        xs = torch.empty((nsamp,) + tuple(x0.shape), dtype=torch.float64, device=x0.device)
        vs = torch.empty_like(xs)
    return x, v, xs, vs


def validate_parameters(m, C, *, stream=None):
    """OscillatorSystem's rule (oscillator.py:75-80) for whole batches: every
    mass and spring rate positive and finite -- the C ABI's own check
    (osc_validate_parameters: one device pass), raising
    NonPositiveParameterError for the first offender (masses first).  The
    integrate entry points run the same check themselves; callers that
    validated once pass ``validate=False`` (OSC_TRUSTED) afterwards."""
    m, C = _dev(m), _dev(C)
    if m.shape != C.shape:
        raise ValueError(f"masses {tuple(m.shape)} vs springs {tuple(C.shape)}")
    bad = ctypes.c_int64(-1)
    rc = _native.lib().osc_validate_parameters(_ptr(m), _ptr(C), m.numel(), ctypes.byref(bad),
                                               ctypes.c_void_p(_stream(stream)))
    raise_for(rc, "osc_validate_parameters", (m, C))


def _energies(nsteps, stride, B, device, want):
    if not want:
        return None
    return torch.empty((1 + nsteps // stride, B), dtype=torch.float64, device=device)


def integrate_batch2(m, C, x0, v0, dt, nsteps, stride=None, *, sample=False, energies=False,
                     compare=False, analytic=None, fma=False, validate=True, stream=None,
                     check=True, t0=0.0) -> BatchResult:
    """Independent 2-DOF systems, SoA ``[2][B]`` (oscillator.py:194-263 for s = 2).

    ``validate`` applies OscillatorSystem's parameter rule to the batch (one
    device reduction; pass False when the same arrays were validated before).
    ``compare``: also return ``errors``, modal.compare of every retained
    sample against the analytic solution (``analytic``: a precomputed
    ``analytic_batch2`` result).  Without samples or energies the error is
    accumulated inside the time loop and no sample is written."""
    lib = _native.lib()
    stride = nsteps if stride is None else stride
    m, C, x0, v0 = (_dev(a) for a in (m, C, x0, v0))
    if m.dim() != 2 or m.shape[0] != 2 or not (m.shape == C.shape == x0.shape == v0.shape):
        raise ValueError(f"expected [2][B] arrays, got {tuple(m.shape)}")
    B = m.shape[1]
    flags = (_native.OSC_FMA if fma else 0) | (0 if validate else _native.OSC_TRUSTED)
    fb = torch.zeros(B, dtype=torch.int64, device=m.device)
    errors = None
    if compare:
        if analytic is None:  # osc_analytic_batch2 applies the parameter rule itself
            sol = analytic_batch2(m, C, x0, v0, stream=stream)
            flags |= _native.OSC_TRUSTED
        else:
            sol = _dev(analytic)
        ts = _dev(accumulated_times(float(t0), float(dt), int(nsteps), int(stride)))
    if compare and not (sample or energies):
        x, v = x0.clone(), v0.clone()
        xs = vs = es = None
        out = torch.empty((3, B), dtype=torch.float64, device=m.device)
        rc = lib.osc_rk4_batch2_compare(_ptr(m), _ptr(C), _ptr(x), _ptr(v), B, float(dt),
                                        int(nsteps), int(stride), _ptr(ts), _ptr(sol), _ptr(out),
                                        _ptr(fb), flags, ctypes.c_void_p(_stream(stream)))
        raise_for(rc, "osc_rk4_batch2_compare", (m, C))
        errors = _reports(out)
    else:
        x, v, xs, vs = _outputs(x0, v0, nsteps, stride, sample or compare)
        es = _energies(nsteps, stride, B, m.device, energies)
        rc = lib.osc_rk4_batch2(_ptr(m), _ptr(C), _ptr(x), _ptr(v), B, float(dt), int(nsteps),
                                int(stride), _ptr(xs), _ptr(vs), _ptr(es), _ptr(fb), flags,
                                ctypes.c_void_p(_stream(stream)))
        raise_for(rc, "osc_rk4_batch2", (m, C))
        if compare:
            errors = compare_batch2(sol, xs, ts, stream=stream)
            bad = fb > 0
            for t in (errors.max_abs_error, errors.rmse, errors.at_time):
                t.masked_fill_(bad, float("nan"))
    res = BatchResult(x, v, xs, vs, fb, float(dt), int(nsteps), int(stride), float(t0),
                      energies=es, errors=errors)
    return res.check() if check else res


def integrate_chains(m, C, x0, v0, dt, nsteps, stride=None, *, sample=False, energies=False,
                     halo_steps=0, fma=False, validate=True, stream=None,
                     check=True, t0=0.0) -> BatchResult:
    """B wall-anchored chains of s cells, ``[B][s]`` (oscillator.py:152-263).
    ``t0``: time label of the initial state (resume, as integrate_batch2)."""
    lib = _native.lib()
    stride = nsteps if stride is None else stride
    m, C, x0, v0 = (_dev(a) for a in (m, C, x0, v0))
    if m.dim() == 1:
        m, C, x0, v0 = (a[None] for a in (m, C, x0, v0))
    if not (m.shape == C.shape == x0.shape == v0.shape) or m.dim() != 2:
        raise ValueError(f"expected [B][s] arrays, got {tuple(m.shape)}")
    B, s = m.shape
    x, v, xs, vs = _outputs(x0, v0, nsteps, stride, sample)
    es = _energies(nsteps, stride, B, m.device, energies)
    fb = torch.zeros(B, dtype=torch.int64, device=m.device)
    rc = lib.osc_rk4_chains(_ptr(m), _ptr(C), _ptr(x), _ptr(v), B, s, float(dt), int(nsteps),
                            int(stride), _ptr(xs), _ptr(vs), _ptr(es), _ptr(fb),
                            int(halo_steps),
                            (_native.OSC_FMA if fma else 0) | (0 if validate else _native.OSC_TRUSTED),
                            ctypes.c_void_p(_stream(stream)))
    raise_for(rc, "osc_rk4_chains", (m, C))
    res = BatchResult(x, v, xs, vs, fb, float(dt), int(nsteps), int(stride), float(t0),
                      energies=es)
    return res.check() if check else res


def integrate_chain_sharded(m, C, x0, v0, dt, nsteps, devices, *, halo_steps=0, fma=False):
    """One chain over several GPUs of this process (osc_rk4_chain_sharded):
    host arrays in, final host ``(x, v)`` out, byte-identical to
    ``integrate_chains`` for any device list (ids may repeat).  Raises
    NonFiniteStateError(step) like integrate."""
    lib = _native.lib()
    m, C = (np.ascontiguousarray(a, np.float64) for a in (m, C))
    x, v = (np.array(a, np.float64, order="C") for a in (x0, v0))
    if not (m.shape == C.shape == x.shape == v.shape) or m.ndim != 1:
        raise ValueError("expected four [s] arrays")
    devs = (ctypes.c_int * len(devices))(*devices)
    fb = np.zeros(1, np.int64)
    rc = lib.osc_rk4_chain_sharded(len(devices), devs, m.ctypes.data, C.ctypes.data,
                                   x.ctypes.data, v.ctypes.data, m.size, float(dt), int(nsteps),
                                   int(halo_steps), fb.ctypes.data,
                                   _native.OSC_FMA if fma else 0)
    if rc == _native.OSC_NONFINITE:
        raise NonFiniteStateError(f"integration diverged at step {int(fb[0])}",
                                  step=int(fb[0]))
    raise_for(rc, "osc_rk4_chain_sharded", (m, C))
    return x, v


def chain_plan(B, s, nsteps, halo_steps=0) -> dict:
    """The launch plan integrate_chains uses (osc_chain_plan; no device work)."""
    out = (ctypes.c_int64 * 7)()
    raise_for(_native.load().osc_chain_plan(int(B), int(s), int(nsteps), int(halo_steps), out),
              "osc_chain_plan")
    keys = ("cells_per_thread", "threads", "steps_per_launch", "owned_per_tile", "halo",
            "tiles_per_chain", "launches")
    return dict(zip(keys, (int(v) for v in out)))


def chain_advance(m, C, xin, vin, xout, vout, own_lo, own_hi, dt, nsteps, step0, first_bad,
                  stream=None, fma=False, left=None, right=None, trusted=False, sync=None,
                  tiles=None, div2=None):
    """One temporally blocked launch over a shard buffer (osc_rk4_chain_advance).

    ``left``/``right``: optional ``(x, v, offset, count)`` -- a neighbour's
    next-input buffers (data pointers) that receive our boundary cells from
    the same kernel (the fused halo exchange).  ``sync``: optional
    ``(ready_left, ready_right, counters, period, timeout_ns)`` -- order the
    edge tiles with the neighbours on the device (osc_edge_sync_t).
    ``tiles``: None (all), "interior" or "edges" -- the two subsets whose
    launches together equal one (OSC_TILES_INTERIOR / OSC_TILES_EDGES).
    ``div2``: the shard's two-operation division table (``div2_table(m)``),
    or None for the three-operation division; same bytes."""
    peers = []
    for p in (left, right):
        peers.append(ctypes.byref(_native.Peer(*p)) if p is not None else None)
    es = None
    if sync is not None:
        rl, rr, ctr, period, timeout_ns = sync
        es = _native.EdgeSync((ctypes.c_void_p * 2)(rl, rr), ctr, int(period), int(timeout_ns))
    rc = _native.lib().osc_rk4_chain_advance_div2(
        _ptr(m), _ptr(C), _ptr(xin), _ptr(vin), _ptr(xout), _ptr(vout), m.numel(), int(own_lo),
        int(own_hi), float(dt), int(nsteps), int(step0), _ptr(first_bad), peers[0], peers[1],
        ctypes.byref(es) if es is not None else None, _ptr(div2),
        (_native.OSC_FMA if fma else 0) | (_native.OSC_TRUSTED if trusted else 0)
        | {None: 0, "interior": _native.OSC_TILES_INTERIOR, "edges": _native.OSC_TILES_EDGES}[tiles],
        ctypes.c_void_p(_stream(stream)))
    raise_for(rc, "osc_rk4_chain_advance", (m, C))


def derivative_chains(m, C, x, *, cell_major=False, stream=None) -> torch.Tensor:
    """dvel per cell (oscillator.py:184-191); [B][s] or, cell_major, [s][B]."""
    lib = _native.lib()
    m, C, x = (_dev(a) for a in (m, C, x))
    B, s = (x.shape[1], x.shape[0]) if cell_major else x.shape
    out = torch.empty_like(x)
    rc = lib.osc_derivative(_ptr(m), _ptr(C), _ptr(x), _ptr(out), B, s,
                                      int(cell_major), ctypes.c_void_p(_stream(stream)))
    raise_for(rc, "osc_derivative", (m, C))
    return out


def energy_chains(m, C, x, v, *, cell_major=False, stream=None) -> torch.Tensor:
    """Exact sequential energy per chain (oscillator.py:266-276) -> [B]."""
    lib = _native.lib()
    m, C, x, v = (_dev(a) for a in (m, C, x, v))
    B, s = (x.shape[1], x.shape[0]) if cell_major else x.shape
    out = torch.empty(B, dtype=torch.float64, device=x.device)
    rc = lib.osc_energy(_ptr(m), _ptr(C), _ptr(x), _ptr(v), _ptr(out), B, s,
                                  int(cell_major), ctypes.c_void_p(_stream(stream)))
    raise_for(rc, "osc_energy", (m, C))
    return out


def check_division(n: int, seed: int = 1, mode: int = 0) -> int:
    """Bitwise mismatches of the hoisted-reciprocal division vs div.rn.f64."""
    out = ctypes.c_uint64(0)
    rc = _native.lib().osc_check_division(int(n), int(seed), int(mode), ctypes.byref(out),
                                          ctypes.c_void_p(_stream()))
    raise_for(rc, "osc_check_division")
    return int(out.value)


def div2_classify(b, *, stream=None) -> torch.Tensor:
    """uint8 tensor of divisor classes for the two-operation division
    (osc_device.cuh div2_classify): 0 = none, 1-3 = admitted (zl itself, or
    moved one ulp toward +inf / -inf).  osc_rk4_batch2 uses it for systems
    whose two masses both have a class."""
    b = _dev(b)
    out = torch.empty(b.numel(), dtype=torch.uint8, device=b.device)
    rc = _native.lib().osc_div2_classify(_ptr(b), b.numel(), _ptr(out),
                                         ctypes.c_void_p(_stream(stream)))
    raise_for(rc, "osc_div2_classify")
    return out.reshape(b.shape)


def div2_table(m, *, stream=None):
    """The 3n-word table [zh | zl | bad] osc_rk4_chain_advance_div2 and
    osc_shard_t.div2 take for a shard's masses m (n cells), or None when
    OSC_DIV2=0 (three-operation division, A/B timing)."""
    if os.environ.get("OSC_DIV2", "1").startswith("0"):
        return None
    m = _dev(m)
    n = m.numel()
    t = torch.empty(3 * n, dtype=torch.float64, device=m.device)
    rc = _native.lib().osc_div2c_table(_ptr(m), n, _ptr(t), _ptr(t[n:]), _ptr(t[2 * n:]),
                                       ctypes.c_void_p(_stream(stream)))
    raise_for(rc, "osc_div2c_table")
    return t


def div2c_table(b, *, stream=None):
    """(zh, zl, bad) of the chain kernels' checked two-operation division
    (osc_device.cuh div2_checked_consts; zh == 0: not eligible)."""
    b = _dev(b)
    zh = torch.empty(b.numel(), dtype=torch.float64, device=b.device)
    zl = torch.empty_like(zh)
    bad = torch.empty(b.numel(), dtype=torch.int64, device=b.device)
    rc = _native.lib().osc_div2c_table(_ptr(b), b.numel(), _ptr(zh), _ptr(zl), _ptr(bad),
                                       ctypes.c_void_p(_stream(stream)))
    raise_for(rc, "osc_div2c_table")
    return zh.reshape(b.shape), zl.reshape(b.shape), bad.reshape(b.shape)


# --------------------------------------------------------------------------
# dense general (M, K) path (BASELINE configs[4]; K5)
# --------------------------------------------------------------------------

def rowscale(K, m, *, stream=None) -> torch.Tensor:
    """A = K / m[:, None] on the device (IEEE division per element)."""
    lib = _native.lib()
    K, m = _dev(K), _dev(m)
    s = m.numel()
    if K.shape != (s, s):
        raise ValueError(f"K must be [{s}][{s}], got {tuple(K.shape)}")
    A = torch.empty_like(K)
    raise_for(lib.osc_rowscale(_ptr(K), _ptr(m), _ptr(A), s, ctypes.c_void_p(_stream(stream))),
              "osc_rowscale", (m, m))
    return A


def integrate_dense(A, X0, V0, dt, nsteps, *, stream=None, check=True) -> BatchResult:
    """N trajectories (columns of X0, V0 [s][N]) of x'' = -A x, classical RK4
    with rk4_step's stage structure (oscillator.py:208-231); two fused FP64
    tensor-core GEMMs per step.  Tolerance-equal (GEMM summation order) to
    the restatement oracle.dense_rk4."""
    lib = _native.lib()
    A, X0, V0 = (_dev(a) for a in (A, X0, V0))
    s, N = X0.shape
    if A.shape != (s, s) or V0.shape != X0.shape:
        raise ValueError("expected A [s][s], X0 and V0 [s][N]")
    x, v = X0.clone(), V0.clone()
    fb = torch.zeros(1, dtype=torch.int64, device=A.device)
    rc = lib.osc_rk4_dense(_ptr(A), _ptr(x), _ptr(v), s, N, float(dt), int(nsteps), _ptr(fb),
                           ctypes.c_void_p(_stream(stream)))
    raise_for(rc, "osc_rk4_dense")
    res = BatchResult(x, v, None, None, fb, float(dt), int(nsteps), int(nsteps))
    return res.check() if check else res
