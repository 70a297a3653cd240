"""The paper's thread-per-equation engine on a GPU warp.

``run_equation_engine`` is the counterpart of ``oscbench.run_parallel``
(parallel.py:395-573): one worker per first-order equation (here a lane of a
single warp), double-banked shared state, a barrier between the RK4 phases.
It returns the trajectory (bit-identical to ``integrate``) and the per-step
latencies measured on the device, summarised with :func:`stats` -- a
restatement of the reference's ``timing.stats`` (timing.py:98-122).
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _native
from .batched import _dev, _ptr, _stream, raise_for
from .oscillator import (NonFiniteStateError, PhaseState, Trajectory, _check_dt, _check_lengths,
                         accumulated_times)


@dataclass(frozen=True)
class LatencyStats:
    """Same fields as oscbench.timing.LatencyStats (timing.py:84-95), seconds."""

    count: int
    mean: float
    stddev: float
    min: float
    p50: float
    p90: float
    p99: float
    max: float


def stats(samples) -> LatencyStats:
    """Mean, population stddev, nearest-rank percentiles (timing.py:98-122)."""
    ordered = sorted(samples)
    n = len(ordered)
    if n == 0:
        raise ValueError("no samples")
    mean = math.fsum(ordered) / n
    var = math.fsum((x - mean) ** 2 for x in ordered) / n

    def rank(p):
        return ordered[max(1, math.ceil(p * n)) - 1]

    return LatencyStats(n, mean, math.sqrt(var), ordered[0], rank(0.50), rank(0.90),
                        rank(0.99), ordered[-1])


@dataclass
class EngineRun:
    trajectory: Trajectory
    step_latencies: list      # seconds, post-warmup
    latency: LatencyStats


def run_equation_engine(system, state0, dt, nsteps, stride=1, warmup=0) -> EngineRun:
    """Integrate on one warp, lanes as equations; measure every step."""
    if nsteps < 1 or stride < 1:
        raise ValueError("nsteps and stride must be >= 1")
    if not 0 <= warmup < nsteps:
        raise ValueError(f"need 0 <= warmup < nsteps, got {warmup}")
    _check_lengths(system, state0)
    _check_dt(dt)
    lib = _native.lib()
    s = len(system.masses)
    m, C, x0, v0 = (_dev(np.asarray(a, dtype=np.float64)) for a in
                    (system.masses, system.springs, state0.positions, state0.velocities))
    nsamp = 1 + nsteps // stride
    xs = torch.empty((nsamp, s), dtype=torch.float64, device=m.device)
    vs = torch.empty_like(xs)
    fb = torch.zeros(1, dtype=torch.int64, device=m.device)
    ns = torch.zeros(nsteps, dtype=torch.int64, device=m.device)
    rc = lib.osc_equation_engine(_ptr(m), _ptr(C), _ptr(x0), _ptr(v0), s, float(dt),
                                 int(nsteps), int(stride), _ptr(xs), _ptr(vs), _ptr(fb), _ptr(ns),
                                 ctypes.c_void_p(_stream()))
    raise_for(rc, "osc_equation_engine")
    bad = int(fb.item())
    if bad:
        raise NonFiniteStateError(f"equation engine diverged at step {bad}", step=bad)
    times = accumulated_times(state0.time, dt, nsteps, stride)
    xs, vs = xs.cpu().numpy(), vs.cpu().numpy()
    samples = [state0] + [PhaseState(xs[j], vs[j], times[j]) for j in range(1, nsamp)]
    lat = (ns.cpu().numpy()[warmup:] * 1e-9).tolist()
    return EngineRun(Trajectory(tuple(samples), dt, stride), lat, stats(lat))
