"""Drop-in mirror of ``oscbench.oscillator`` whose arithmetic runs on the B200.

Same names, argument meaning, validation order, return types and exceptions
as ``/root/reference/pkg/src/oscbench/oscillator.py``; the time stepping
(``integrate``, ``rk4_step``) and the per-cell operations (``derivative``,
``energy``) execute as sm_100a kernels through ``libosc_b200.so``.  Results are
byte-identical to the reference (tests/test_gpu_parity.py).

The functions accept the reference's own objects too (anything with
``masses``/``springs`` and ``positions``/``velocities``/``time``), so
``oscbench`` callers can switch by rebinding ``integrate``.
"""

from __future__ import annotations

import math
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


def _check_lengths(system, state):
    """oscillator.py:177-181."""
    if len(state.positions) != len(system.masses):
        raise LengthMismatchError(
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


def integrate(system, state0, dt: float, nsteps: int, stride: int = 1) -> Trajectory:
    """Fixed-step RK4 integration on the GPU (oscillator.py:234-263).

    Retains the initial state plus every ``stride``-th state.  Raises
    ``NonFiniteStateError`` with ``.step`` = the first diverging step.
    """
    from . import batched

    if nsteps < 1:
        raise ValueError(f"nsteps must be >= 1, got {nsteps}")
    if stride < 1:
        raise ValueError(f"stride must be >= 1, got {stride}")
    _check_lengths(system, state0)
    _check_dt(dt)
    s = len(system.masses)
    m = np.asarray(system.masses, dtype=np.float64)
    C = np.asarray(system.springs, dtype=np.float64)
    x0 = np.asarray(state0.positions, dtype=np.float64)
    v0 = np.asarray(state0.velocities, dtype=np.float64)
    if s == 2:
        res = batched.integrate_batch2(m[:, None], C[:, None], x0[:, None], v0[:, None], dt,
                                       nsteps, stride, sample=True, check=False)
        xs = res.xs[..., 0].cpu().numpy()
        vs = res.vs[..., 0].cpu().numpy()
    else:
        res = batched.integrate_chains(m[None], C[None], x0[None], v0[None], dt, nsteps, stride,
                                       sample=True, check=False)
        xs = res.xs[:, 0].cpu().numpy()
        vs = res.vs[:, 0].cpu().numpy()
    bad = int(res.first_bad.max().item())
    if bad:
        raise NonFiniteStateError(f"integration diverged at step {bad}: non-finite phase entry",
                                  step=bad)
    times = accumulated_times(state0.time, dt, nsteps, stride)
    samples = [state0] + [PhaseState(xs[j], vs[j], times[j]) for j in range(1, len(times))]
    return Trajectory(tuple(samples), dt, stride)


def rk4_step(system, state, dt: float) -> PhaseState:
    """One classical RK4 step on the GPU (oscillator.py:194-231)."""
    _check_dt(dt)
    _check_lengths(system, state)
    traj = integrate_arrays(system, state, dt)
    x, v, bad = traj
    if bad:
        bad_vals = [u for u in np.concatenate([x, v]) if not math.isfinite(u)] or [math.nan]
        raise NonFiniteStateError(f"non-finite phase entry {bad_vals[0]!r}")
    return PhaseState(x, v, state.time + dt)


def integrate_arrays(system, state, dt: float, nsteps: int = 1):
    """Final (x, v, first_bad) after nsteps, no sampling (host numpy arrays)."""
    from . import batched

    m = np.asarray(system.masses, dtype=np.float64)
    C = np.asarray(system.springs, dtype=np.float64)
    x0 = np.asarray(state.positions, dtype=np.float64)
    v0 = np.asarray(state.velocities, dtype=np.float64)
    res = batched.integrate_chains(m[None], C[None], x0[None], v0[None], dt, nsteps, nsteps,
                                   sample=False, check=False)
    return res.x[0].cpu().numpy(), res.v[0].cpu().numpy(), int(res.first_bad[0].item())


def derivative(system, state) -> PhaseDerivative:
    """dpos = velocities, dvel = acceleration_at per cell (oscillator.py:184-191)."""
    from . import batched

    _check_lengths(system, state)
    dvel = batched.derivative_chains(
        np.asarray(system.masses, dtype=np.float64)[None],
        np.asarray(system.springs, dtype=np.float64)[None],
        np.asarray(state.positions, dtype=np.float64)[None])
    return PhaseDerivative(state.velocities, dvel[0].cpu().numpy())


def energy(system, state) -> float:
    """Total mechanical energy, sequential sum (oscillator.py:266-276)."""
    from . import batched

    _check_lengths(system, state)
    out = batched.energy_chains(
        np.asarray(system.masses, dtype=np.float64)[None],
        np.asarray(system.springs, dtype=np.float64)[None],
        np.asarray(state.positions, dtype=np.float64)[None],
        np.asarray(state.velocities, dtype=np.float64)[None])
    return float(out[0].item())
