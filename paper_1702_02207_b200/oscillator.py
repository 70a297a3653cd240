"""Drop-in mirror of ``oscbench.oscillator`` whose arithmetic runs on the B200.

Same names, argument meaning, validation order, return types and exceptions
as ``/root/reference/pkg/src/oscbench/oscillator.py``; the time stepping
(``integrate``, ``rk4_step``) and the per-cell operations (``derivative``,
``energy``) execute as sm_100a kernels through ``libosc_b200.so``.  Results are
byte-identical to the reference (tests/test_gpu_parity.py).

The functions accept the reference's own objects too (anything with
``masses``/``springs`` and ``positions``/``velocities``/``time``), so
``oscbench`` callers can switch by rebinding ``integrate`` (INTEGRATION.md,
:mod:`.dropin`).  Results come back in the caller's type family: given the
reference's ``PhaseState``, ``integrate`` returns the reference's
``Trajectory`` of reference ``PhaseState`` objects, and every error it raises
is an instance of BOTH the reference's class and ours (:func:`_family`), so
``except oscbench.NonFiniteStateError`` keeps working after the rebinding.
"""

from __future__ import annotations

import math
import sys
from dataclasses import dataclass

import numpy as np

__all__ = [
    "NonPositiveParameterError",
    "LengthMismatchError",
    "NonFiniteStateError",
    "DimensionMismatchError",
    "OscillatorSystem",
    "PhaseState",
    "PhaseDerivative",
    "Trajectory",
    "build_chain",
    "derivative",
    "rk4_step",
    "integrate",
    "energy",
]


class NonPositiveParameterError(ValueError):
    """A mass or spring rate is zero, negative, or non-finite (oscillator.py:39-40)."""


class LengthMismatchError(ValueError):
    """Vector lengths disagree with the system's size (oscillator.py:43-44)."""


class NonFiniteStateError(ArithmeticError):
    """Integration produced a NaN or infinity (oscillator.py:47-52)."""

    def __init__(self, message: str, step: int | None = None):
        super().__init__(message)
        self.step = step


class DimensionMismatchError(ValueError):
    """Operation is defined only for a two-mass chain (oscillator.py:55-56)."""


@dataclass(frozen=True)
class OscillatorSystem:
    """Validated wall-anchored chain (oscillator.py:59-84)."""

    masses: tuple[float, ...]
    springs: tuple[float, ...]

    def __post_init__(self):
        object.__setattr__(self, "masses", tuple(float(m) for m in self.masses))
        object.__setattr__(self, "springs", tuple(float(c) for c in self.springs))
        if not self.masses:
            raise NonPositiveParameterError("chain needs at least one mass")
        if len(self.masses) != len(self.springs):
            raise LengthMismatchError(f"{len(self.masses)} masses vs {len(self.springs)} springs")
        for label, values in (("masses", self.masses), ("springs", self.springs)):
            for i, v in enumerate(values):
                if not math.isfinite(v) or v <= 0.0:
                    raise NonPositiveParameterError(
                        f"{label}[{i}] = {v!r}; must be positive and finite")

    @property
    def size(self) -> int:
        return len(self.masses)


def build_chain(masses, springs) -> OscillatorSystem:
    """oscillator.py:87-89."""
    return OscillatorSystem(tuple(masses), tuple(springs))


@dataclass(frozen=True)
class PhaseState:
    """Positions, velocities and elapsed time (oscillator.py:92-113)."""

    positions: tuple[float, ...]
    velocities: tuple[float, ...]
    time: float = 0.0

    def __post_init__(self):
        object.__setattr__(self, "positions", tuple(float(x) for x in self.positions))
        object.__setattr__(self, "velocities", tuple(float(v) for v in self.velocities))
        if len(self.positions) != len(self.velocities):
            raise LengthMismatchError(
                f"{len(self.positions)} positions vs {len(self.velocities)} velocities")
        for v in self.positions + self.velocities:
            if not math.isfinite(v):
                raise NonFiniteStateError(f"non-finite phase entry {v!r}")

    @property
    def size(self) -> int:
        return len(self.positions)


@dataclass(frozen=True)
class PhaseDerivative:
    """dpos in m/s, dvel in m/s^2 (oscillator.py:116-130)."""

    dpos: tuple[float, ...]
    dvel: tuple[float, ...]

    def __post_init__(self):
        object.__setattr__(self, "dpos", tuple(float(x) for x in self.dpos))
        object.__setattr__(self, "dvel", tuple(float(v) for v in self.dvel))
        if len(self.dpos) != len(self.dvel):
            raise LengthMismatchError("dpos/dvel length mismatch")
        for v in self.dpos + self.dvel:
            if not math.isfinite(v):
                raise NonFiniteStateError(f"non-finite derivative entry {v!r}")


@dataclass(frozen=True)
class Trajectory:
    """States retained every ``stride`` steps, initial first (oscillator.py:133-149)."""

    samples: tuple[PhaseState, ...]
    dt: float
    stride: int

    def __post_init__(self):
        object.__setattr__(self, "samples", tuple(self.samples))

    @property
    def final_state(self) -> PhaseState:
        return self.samples[-1]

    def times(self) -> list[float]:
        return [s.time for s in self.samples]


class _Family:
    """The types one call returns and raises: ours, or a foreign module's
    (the reference's ``oscbench.oscillator``) bridged to ours."""

    NAMES = ("PhaseState", "PhaseDerivative", "Trajectory")
    ERRORS = ("NonFiniteStateError", "LengthMismatchError", "NonPositiveParameterError",
              "DimensionMismatchError")

    def __init__(self, mod):
        own = sys.modules[__name__]
        for name in self.NAMES:
            setattr(self, name, getattr(mod, name))
        for name in self.ERRORS:
            ours, theirs = getattr(own, name), getattr(mod, name, None)
            if theirs is None or theirs is ours:
                setattr(self, name, ours)
            else:
                # caught by `except oscbench.X` and by `except paper_1702_02207_b200.X`
                setattr(self, name, type(name, (ours, theirs), {"__module__": mod.__name__}))


_FAMILIES: dict = {}


def _family(*objs) -> _Family:
    """The type family of the first argument built from a foreign module that
    defines the reference's public types (e.g. ``oscbench.oscillator``); ours
    otherwise."""
    own = sys.modules[__name__]
    for obj in objs:
        mod = sys.modules.get(type(obj).__module__)
        if mod is None or mod is own:
            continue
        if all(hasattr(mod, n) for n in _Family.NAMES + ("NonFiniteStateError",)):
            fam = _FAMILIES.get(mod.__name__)
            if fam is None or fam.PhaseState is not mod.PhaseState:
                fam = _FAMILIES[mod.__name__] = _Family(mod)
            return fam
    fam = _FAMILIES.get(__name__)
    if fam is None:
        fam = _FAMILIES[__name__] = _Family(own)
    return fam


def _check_lengths(system, state, fam=None):
    """oscillator.py:177-181."""
    if len(state.positions) != len(system.masses):
        raise (fam or _family(state, system)).LengthMismatchError(
            f"state has {len(state.positions)} coordinates, system has {len(system.masses)}")


def _check_dt(dt):
    """rk4_step's dt rule (oscillator.py:201-202)."""
    if not (isinstance(dt, (int, float)) and math.isfinite(dt) and dt > 0.0):
        raise ValueError(f"dt must be positive and finite, got {dt!r}")


def accumulated_times(t0: float, dt: float, nsteps: int, stride: int) -> np.ndarray:
    """Labels of the retained samples: ``t += dt`` once per step, in order.

    The reference labels each state with ``state.time + dt`` (oscillator.py:231),
    a sequential sum, not ``k*dt``.  ``np.add.accumulate`` is a left fold, so
    it reproduces that sum bit for bit; chunks bound the memory.
    """
    out = [float(t0)]
    t = float(t0)
    chunk = 1 << 20
    k = 0
    while k < nsteps:
        n = min(chunk, nsteps - k)
        run = np.add.accumulate(np.concatenate(([t], np.full(n, float(dt)))))
        steps = np.arange(k + 1, k + n + 1)
        out.extend(run[1:][steps % stride == 0].tolist())
        t = float(run[-1])
        k += n
    return np.array(out)


def _first_nonfinite(x, v) -> float:
    """The entry PhaseState.__post_init__ names (oscillator.py:107-109):
    the first non-finite of positions + velocities."""
    for u in np.concatenate([np.asarray(x, dtype=np.float64), np.asarray(v, dtype=np.float64)]):
        if not math.isfinite(u):
            return float(u)
    return math.nan


def _host_run(system, state, dt, nsteps, stride, sample):
    """One system through the host-pointer C ABI (osc_rk4_batch2_host for
    two masses, osc_rk4_chains_host otherwise): numpy in, numpy out, one
    staged round trip for small systems.  Returns (x, v, xs, vs, first_bad)
    with xs/vs [1 + nsteps // stride][s] when ``sample``."""
    from . import _native
    from .batched import raise_for

    lib = _native.lib()
    m = np.ascontiguousarray(system.masses, dtype=np.float64)
    C = np.ascontiguousarray(system.springs, dtype=np.float64)
    x = np.array(state.positions, dtype=np.float64)
    v = np.array(state.velocities, dtype=np.float64)
    s = x.size
    nsamp = 1 + nsteps // stride
    xs = np.empty((nsamp, s)) if sample else None
    vs = np.empty((nsamp, s)) if sample else None
    fb = np.zeros(1, dtype=np.int64)
    ptr = lambda a: None if a is None else a.ctypes.data  # noqa: E731
    if s == 2:  # [2][B] with B = 1 is the same memory as [2]
        rc = lib.osc_rk4_batch2_host(ptr(m), ptr(C), ptr(x), ptr(v), 1, float(dt), int(nsteps),
                                     int(stride), ptr(xs), ptr(vs), ptr(fb))
    else:
        rc = lib.osc_rk4_chains_host(ptr(m), ptr(C), ptr(x), ptr(v), 1, s, float(dt),
                                     int(nsteps), int(stride), ptr(xs), ptr(vs), ptr(fb))
    if rc != _native.OSC_NONFINITE:
        raise_for(rc, "integrate", (m, C))
    return x, v, xs, vs, int(fb[0])


def integrate(system, state0, dt: float, nsteps: int, stride: int = 1) -> Trajectory:
    """Fixed-step RK4 integration on the GPU (oscillator.py:234-263).

    Retains the initial state plus every ``stride``-th state.  Raises
    ``NonFiniteStateError`` with ``.step`` = the first diverging step and the
    reference's message (the first non-finite entry of the state at that
    step, recomputed exactly by a second run of ``step`` steps).
    """
    if nsteps < 1:
        raise ValueError(f"nsteps must be >= 1, got {nsteps}")
    if stride < 1:
        raise ValueError(f"stride must be >= 1, got {stride}")
    fam = _family(state0, system)
    _check_lengths(system, state0, fam)
    _check_dt(dt)
    _, _, xs, vs, bad = _host_run(system, state0, dt, nsteps, stride, True)
    if bad:
        xb, vb, _ = integrate_arrays(system, state0, dt, bad)
        raise fam.NonFiniteStateError(
            f"integration diverged at step {bad}: non-finite phase entry "
            f"{_first_nonfinite(xb, vb)!r}", step=bad)
    times = accumulated_times(state0.time, dt, nsteps, stride)
    make = fam.PhaseState
    samples = [state0] + [make(xs[j], vs[j], times[j]) for j in range(1, len(times))]
    return fam.Trajectory(tuple(samples), dt, stride)


def rk4_step(system, state, dt: float) -> PhaseState:
    """One classical RK4 step on the GPU (oscillator.py:194-231)."""
    _check_dt(dt)
    fam = _family(state, system)
    _check_lengths(system, state, fam)
    x, v, bad = integrate_arrays(system, state, dt)
    if bad:
        raise fam.NonFiniteStateError(f"non-finite phase entry {_first_nonfinite(x, v)!r}")
    return fam.PhaseState(x, v, state.time + dt)


def integrate_arrays(system, state, dt: float, nsteps: int = 1):
    """Final (x, v, first_bad) after nsteps, no sampling (host numpy arrays)."""
    x, v, _, _, bad = _host_run(system, state, dt, nsteps, nsteps, False)
    return x, v, bad


def derivative(system, state) -> PhaseDerivative:
    """dpos = velocities, dvel = acceleration_at per cell (oscillator.py:184-191),
    one staged round trip through osc_derivative_host."""
    from . import _native
    from .batched import raise_for

    fam = _family(state, system)
    _check_lengths(system, state, fam)
    lib = _native.lib()
    m = np.ascontiguousarray(system.masses, dtype=np.float64)
    C = np.ascontiguousarray(system.springs, dtype=np.float64)
    x = np.ascontiguousarray(state.positions, dtype=np.float64)
    dvel = np.empty_like(x)
    rc = lib.osc_derivative_host(m.ctypes.data, C.ctypes.data, x.ctypes.data, dvel.ctypes.data,
                                 1, x.size, 0)
    raise_for(rc, "derivative", (m, C))
    if not np.isfinite(dvel).all():
        raise fam.NonFiniteStateError(
            f"non-finite derivative entry {_first_nonfinite(state.velocities, dvel)!r}")
    return fam.PhaseDerivative(state.velocities, dvel)


def energy(system, state) -> float:
    """Total mechanical energy, sequential sum (oscillator.py:266-276), one
    staged round trip through osc_energy_host."""
    from . import _native
    from .batched import raise_for

    _check_lengths(system, state)
    lib = _native.lib()
    m = np.ascontiguousarray(system.masses, dtype=np.float64)
    C = np.ascontiguousarray(system.springs, dtype=np.float64)
    x = np.ascontiguousarray(state.positions, dtype=np.float64)
    v = np.ascontiguousarray(state.velocities, dtype=np.float64)
    out = np.empty(1)
    rc = lib.osc_energy_host(m.ctypes.data, C.ctypes.data, x.ctypes.data, v.ctypes.data,
                             out.ctypes.data, 1, x.size, 0)
    raise_for(rc, "energy", (m, C))
    return float(out[0])
