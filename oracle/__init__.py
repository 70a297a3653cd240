"""TEST INFRASTRUCTURE ONLY -- CPU oracle for the RK4 hot path.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference``) may import this package, and
only as the checker / the timed CPU baseline.  The product package
``paper_1702_02207_b200`` never imports it; its CUDA path fails loudly when
the extension is missing.

Three restatements of the reference integrator
``/root/reference/pkg/src/oscbench/oscillator.py`` live here:

* ``liboracle.so`` (``rk4_oracle.c``): a plain-C restatement, OpenMP over
  independent chains or over cells inside each RK4 phase.  Byte-identical to
  ``oscbench.integrate`` (``-ffp-contract=off``).
* ``np_*``: numpy restatements, vectorised over cells/systems.  Elementwise
  IEEE operations in the reference's order; numpy never fuses a*b+c, so these
  are byte-identical too.
* ``dense_*``: the dense general-(M,K) restatement (no reference symbol; the
  reference keeps only the chain) and its eigen-analytic
  solution.

Parity is pinned: ``tests/test_oracle.py`` checks every restatement against
``tests/golden/*.npz``, which ``tests/golden/gen_golden.py`` produced by
running the reference package itself.
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None

_i64 = ctypes.c_int64
_dp = ctypes.POINTER(ctypes.c_double)
_ip = ctypes.POINTER(ctypes.c_int64)


def build() -> str:
    """Compile liboracle.so with the committed Makefile (no reference build)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return os.path.join(_HERE, "liboracle.so")


def lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "liboracle.so")
        if not os.path.exists(path):
            build()
        L = ctypes.CDLL(path)
        L.oracle_rk4_chains.restype = ctypes.c_int
        L.oracle_rk4_chains.argtypes = [_dp, _dp, _dp, _dp, _i64, _i64, ctypes.c_double,
                                        _i64, _i64, _dp, _dp, _ip, ctypes.c_int]
        L.oracle_rk4_chain_mt.restype = ctypes.c_int
        L.oracle_rk4_chain_mt.argtypes = [_dp, _dp, _dp, _dp, _i64, ctypes.c_double, _i64,
                                          _ip, ctypes.c_int]
        L.oracle_rk4_batch2.restype = ctypes.c_int
        L.oracle_rk4_batch2.argtypes = [_dp, _dp, _dp, _dp, _i64, ctypes.c_double, _i64, _ip,
                                        ctypes.c_int]
        L.oracle_energy.restype = None
        L.oracle_energy.argtypes = [_dp, _dp, _dp, _dp, _i64, _i64, _dp]
        L.oracle_derivative.restype = None
        L.oracle_derivative.argtypes = [_dp, _dp, _dp, _i64, _i64, _dp]
        _LIB = L
    return _LIB


def _p(a):
    return a.ctypes.data_as(_dp) if a is not None else None


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


# --------------------------------------------------------------------------
# C restatement
# --------------------------------------------------------------------------

def c_rk4_chains(m, C, x0, v0, dt, nsteps, stride=None, sample=True, nthreads=0):
    """integrate() for B chains laid out [B][s] (oscillator.py:234-263).

    Returns ``(xs, vs, x, v, first_bad)``: samples ``[1+nsteps//stride][B][s]``
    (None when ``sample`` is false), final state ``[B][s]`` and the 1-based
    first non-finite step per chain (0 = none).
    """
    m, C = _f64(m), _f64(C)
    x, v = _f64(x0).copy(), _f64(v0).copy()
    B, s = x.shape
    stride = nsteps if stride is None else stride
    xs = vs = None
    if sample:
        nsamp = 1 + nsteps // stride
        xs = np.full((nsamp, B, s), np.nan)
        vs = np.full((nsamp, B, s), np.nan)
    fb = np.zeros(B, dtype=np.int64)
    rc = lib().oracle_rk4_chains(_p(m), _p(C), _p(x), _p(v), B, s, float(dt), int(nsteps),
                                 int(stride), _p(xs), _p(vs),
                                 fb.ctypes.data_as(_ip), int(nthreads))
    if rc < 0:
        raise MemoryError("oracle scratch allocation failed")
    return xs, vs, x, v, fb


def c_rk4_batch2(m, C, x0, v0, dt, nsteps, stride=None, sample=True, nthreads=0):
    """Batched 2-DOF systems in the product's SoA layout ``[2][B]``."""
    T = lambda a: _f64(a).T.copy()
    xs, vs, x, v, fb = c_rk4_chains(T(m), T(C), T(x0), T(v0), dt, nsteps, stride,
                                    sample, nthreads)
    if xs is not None:
        xs = np.ascontiguousarray(xs.transpose(0, 2, 1))
        vs = np.ascontiguousarray(vs.transpose(0, 2, 1))
    return xs, vs, x.T.copy(), v.T.copy(), fb


def c_rk4_batch2_final(m, C, x0, v0, dt, nsteps, nthreads=0):
    """Batched 2-DOF, SoA [2][B], final state only (register-resident form)."""
    m, C = _f64(m), _f64(C)
    x, v = _f64(x0).copy(), _f64(v0).copy()
    B = x.shape[1]
    fb = np.zeros(B, dtype=np.int64)
    lib().oracle_rk4_batch2(_p(m), _p(C), _p(x), _p(v), B, float(dt), int(nsteps),
                            fb.ctypes.data_as(_ip), int(nthreads))
    return x, v, fb


def c_rk4_chain_mt(m, C, x0, v0, dt, nsteps, nthreads=0):
    """One long chain, cells split across threads in every phase."""
    m, C = _f64(m), _f64(C)
    x, v = _f64(x0).copy(), _f64(v0).copy()
    fb = np.zeros(1, dtype=np.int64)
    lib().oracle_rk4_chain_mt(_p(m), _p(C), _p(x), _p(v), x.shape[0], float(dt),
                              int(nsteps), fb.ctypes.data_as(_ip), int(nthreads))
    return x, v, int(fb[0])


def c_energy(m, C, x, v):
    m, C, x, v = (np.atleast_2d(_f64(a)) for a in (m, C, x, v))
    B, s = x.shape
    out = np.empty(B)
    lib().oracle_energy(_p(m), _p(C), _p(x), _p(v), B, s, _p(out))
    return out


def c_derivative(m, C, x):
    m, C, x = (np.atleast_2d(_f64(a)) for a in (m, C, x))
    B, s = x.shape
    out = np.empty((B, s))
    lib().oracle_derivative(_p(m), _p(C), _p(x), B, s, _p(out))
    return out


# --------------------------------------------------------------------------
# numpy restatement (vectorised over the last axis = cells)
# --------------------------------------------------------------------------

def np_accel(m, C, x):
    """acceleration_at (oscillator.py:152-164) for all cells at once.

    left_i = x_i - x_{i-1} (x_{-1} = wall; x_0 - 0.0 == x_0 exactly),
    a = (-C_i)*left_i  [= -(C_i*left_i) exactly under round-to-nearest],
    a += C_{i+1}*(x_{i+1}-x_i) for i < s-1, then a / m_i.
    """
    d = np.empty_like(x)
    d[..., 0] = x[..., 0] - 0.0
    d[..., 1:] = x[..., 1:] - x[..., :-1]
    a = (-C) * d
    a[..., :-1] = a[..., :-1] + C[..., 1:] * d[..., 1:]
    return a / m


def np_rk4_step(m, C, pos, vel, dt):
    """rk4_step (oscillator.py:194-231), arrays [..., s]."""
    half_dt = 0.5 * dt
    k1v = np_accel(m, C, pos)
    y2p = pos + half_dt * vel
    y2v = vel + half_dt * k1v
    k2v = np_accel(m, C, y2p)
    y3p = pos + half_dt * y2v
    y3v = vel + half_dt * k2v
    k3v = np_accel(m, C, y3p)
    y4p = pos + dt * y3v
    y4v = vel + dt * k3v
    k4v = np_accel(m, C, y4p)
    dt6 = dt / 6.0
    new_pos = pos + dt6 * (vel + 2.0 * y2v + 2.0 * y3v + y4v)
    new_vel = vel + dt6 * (k1v + 2.0 * k2v + 2.0 * k3v + k4v)
    return new_pos, new_vel


def np_integrate(m, C, x0, v0, dt, nsteps, stride=1):
    """integrate (oscillator.py:234-263) over arrays [..., s].

    Returns ``(xs, vs, first_bad)`` with samples ``[1+nsteps//stride, ..., s]``;
    ``first_bad`` is the 1-based step at which any cell of the batch first
    turned non-finite (0 = never); sampling stops there, as the reference
    raises at that step.
    """
    m, C = _f64(m), _f64(C)
    pos, vel = _f64(x0), _f64(v0)
    xs, vs = [pos.copy()], [vel.copy()]
    for k in range(nsteps):
        with np.errstate(all="ignore"):  # divergence is detected below, as the reference does
            pos, vel = np_rk4_step(m, C, pos, vel, dt)
        if not (np.isfinite(pos).all() and np.isfinite(vel).all()):
            return np.array(xs), np.array(vs), k + 1
        if (k + 1) % stride == 0:
            xs.append(pos.copy())
            vs.append(vel.copy())
    return np.array(xs), np.array(vs), 0


def light_cone(s, a, b, nsteps):
    """Window [a,b) of a chain after nsteps depends on [a-2n, b+2n) only.

    Dependency radius is 2 cells of x and v per RK4 step.  Returns
    ``(lo, hi, off)``: simulate cells [lo,hi) as their own chain (wall-left,
    free-right: exact when lo == 0 / hi == s) and read cells
    [off, off + (b-a)) of the result.
    """
    lo = max(0, a - 2 * nsteps)
    hi = min(s, b + 2 * nsteps)
    return lo, hi, a - lo


# --------------------------------------------------------------------------
# analytic two-mode oracle: restatement of oscbench/modal.py
# --------------------------------------------------------------------------

_SQRT5 = math.sqrt(5.0)


def characteristic_frequencies(m, c):
    """modal.py:76-82."""
    return (math.sqrt(c * (3.0 + _SQRT5) / (2.0 * m)),
            math.sqrt(c * (3.0 - _SQRT5) / (2.0 * m)))


def mode_ratios(m, c):
    """modal.py:85-95."""
    w1, w2 = characteristic_frequencies(m, c)
    return 2.0 - m * (w1 * w1) / c, 2.0 - m * (w2 * w2) / c


def analytic_solution(m, c, x0, v0):
    """modal.py:98-120 -> (omega1, omega2, r1, r2, a1c, a1s, a2c, a2s)."""
    w1, w2 = characteristic_frequencies(m, c)
    r1, r2 = mode_ratios(m, c)
    det = r2 - r1
    a1c = (r2 * x0[0] - x0[1]) / det
    a2c = (x0[1] - r1 * x0[0]) / det
    u1 = (r2 * v0[0] - v0[1]) / det
    u2 = (v0[1] - r1 * v0[0]) / det
    return (w1, w2, r1, r2, a1c, u1 / w1, a2c, u2 / w2)


def eval_analytic(sol, t):
    """modal.py:123-129, vectorised over t."""
    w1, w2, r1, r2, a1c, a1s, a2c, a2s = sol
    t = np.asarray(t, dtype=np.float64)
    mode1 = a1c * np.cos(w1 * t) + a1s * np.sin(w1 * t)
    mode2 = a2c * np.cos(w2 * t) + a2s * np.sin(w2 * t)
    return mode1 + mode2, r1 * mode1 + r2 * mode2


def compare(times, xs, sol):
    """modal.py:141-162: (max |err|, rmse, at_time) over both coordinates.

    ``xs`` is ``[nsamp][2]`` positions, ``times`` the accumulated labels.
    """
    x1a, x2a = eval_analytic(sol, times)
    err = np.abs(np.stack([xs[:, 0] - x1a, xs[:, 1] - x2a], axis=1))
    flat = err.reshape(-1)
    j = int(np.argmax(flat))
    return float(flat[j]), float(math.sqrt(np.mean(flat * flat))), float(times[j // 2])


def compare_seq(times, xs, sol):
    """modal.py:141-162 literally: samples in order, both coordinates,
    sequential sum of squares, strict ``>`` for the maximum.  math.cos/sin
    (glibc) as in the reference.  -> (max_abs_error, rmse, at_time)."""
    w1, w2, r1, r2, a1c, a1s, a2c, a2s = (float(f) for f in sol)
    max_err, at_time, sum_sq, count = -1.0, 0.0, 0.0, 0
    for t, (p0, p1) in zip(times, xs):
        t = float(t)
        mode1 = a1c * math.cos(w1 * t) + a1s * math.sin(w1 * t)
        mode2 = a2c * math.cos(w2 * t) + a2s * math.sin(w2 * t)
        for num, ana in ((float(p0), mode1 + mode2), (float(p1), r1 * mode1 + r2 * mode2)):
            err = abs(num - ana)
            sum_sq += err * err
            count += 1
            if err > max_err:
                max_err, at_time = err, t
    return max_err, math.sqrt(sum_sq / count), at_time


def analytic_general(m0, m1, C0, C1, x0, v0):
    """Two-mode solution of a 2-DOF wall-anchored chain with arbitrary
    parameters: analytic_solution (modal.py:98-120) when m0 == m1 and
    C0 == C1, else the same modal construction for K - w^2 M with
    K = [[C0 + C1, -C1], [-C1, C1]], M = diag(m0, m1) -- operation for
    operation what osc_modal.cuh computes (outside the reference)."""
    if m0 == m1 and C0 == C1:
        return analytic_solution(m0, C0, x0, v0)
    a = m0 * m1
    b = m0 * C1 + m1 * (C0 + C1)
    c = C0 * C1
    disc = b * b - 4.0 * (a * c)
    q = b + math.sqrt(disc if disc > 0.0 else 0.0)
    L1 = q / (2.0 * a)
    L2 = (2.0 * c) / q
    w1, w2 = math.sqrt(L1), math.sqrt(L2)
    r1 = C1 / (C1 - L1 * m1)
    r2 = C1 / (C1 - L2 * m1)
    det = r2 - r1
    a1c = (r2 * x0[0] - x0[1]) / det
    a2c = (x0[1] - r1 * x0[0]) / det
    u1 = (r2 * v0[0] - v0[1]) / det
    u2 = (v0[1] - r1 * v0[0]) / det
    return (w1, w2, r1, r2, a1c, u1 / w1, a2c, u2 / w2)


# --------------------------------------------------------------------------
# dense general-(M,K) restatement (SPEC.md:8/188 -- outside the reference)
# --------------------------------------------------------------------------

def dense_rk4(A, X0, V0, dt, nsteps):
    """rk4_step's stage structure (oscillator.py:208-228) with
    acceleration_at replaced by ``-(A @ Y)``, A = M^-1 K.  X0/V0 are [s][N]
    (one trajectory per column).  Returns final (X, V)."""
    A = _f64(A)
    X, V = _f64(X0).copy(), _f64(V0).copy()
    h = 0.5 * dt
    dt6 = dt / 6.0
    for _ in range(nsteps):
        k1 = -(A @ X)
        y2p = X + h * V
        y2v = V + h * k1
        k2 = -(A @ y2p)
        y3p = X + h * y2v
        y3v = V + h * k2
        k3 = -(A @ y3p)
        y4p = X + dt * y3v
        y4v = V + dt * k3
        k4 = -(A @ y4p)
        X, V = (X + dt6 * (V + 2.0 * y2v + 2.0 * y3v + y4v),
                V + dt6 * (k1 + 2.0 * k2 + 2.0 * k3 + k4))
    return X, V


def dense_analytic(m, K, X0, t):
    """Exact x(t) for M x'' + K x = 0, v(0) = 0:
    x(t) = M^-1/2 W cos(sqrt(L) t) W^T M^1/2 x0 with W L W^T = M^-1/2 K M^-1/2."""
    m = _f64(m)
    sm = np.sqrt(m)
    S = K / sm[:, None] / sm[None, :]
    S = 0.5 * (S + S.T)
    lam, W = np.linalg.eigh(S)
    Z = W.T @ (sm[:, None] * _f64(X0))
    Z = np.cos(np.sqrt(lam) * t)[:, None] * Z
    return (W @ Z) / sm[:, None]
