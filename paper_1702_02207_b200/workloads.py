"""Seeded synthetic inputs for the five BASELINE.json configurations.

There is no public dataset for this path: every input is drawn
on the host with numpy ``default_rng(SEED)`` (PCG64) in the draw order below,
so the CPU oracle and the GPU consume identical bits.  Layouts are SoA fp64:

* C1  one paper 2-DOF system (eq. 3), m=1, C=1012.5 (C/m exactly 1012.5).
* C2  ``[2][B]`` batch of independent 2-DOF systems (eq. 2), B = 2**20.
* C3  one wall-anchored chain of s = 2**24 cells.
* C4  ``[B][s]`` batch of 4096 chains of 1024 cells.
* C5  dense s=4096 system, ``A = M^-1 K`` and ``X0`` as ``[s][N]``, N = 1024.

"Fixed ends" in BASELINE.json is read as the reference topology: spring 0
anchors cell 0 to the wall, the last cell is free (oscillator.py:3-5,160-163;
``len(springs) == len(masses)`` leaves no right wall).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

SEED = 170202207  # arXiv 1702.02207

C2_B = 1 << 20
C3_S = 1 << 24
C4_B, C4_S = 4096, 1024
C5_S, C5_N = 4096, 1024


@dataclass(frozen=True)
class RunParams:
    dt: float
    nsteps: int
    stride: int


PARAMS = {
    "C1": RunParams(1e-4, 1_000_000, 1000),
    "C2": RunParams(1e-4, 10_000, 10_000),
    "C3": RunParams(1e-4, 10_000, 10_000),
    "C4": RunParams(1e-4, 10_000, 10_000),
    "C5": RunParams(1e-4, 1000, 1000),
}


def _rng():
    return np.random.default_rng(SEED)


def part(n: int, rank: int, world: int) -> slice:
    """Rank's contiguous share [n*rank//world, n*(rank+1)//world) of n
    independent units (C2 systems, C4 chains, C5 trajectory
    columns) -- a split of the ONE seeded draw, so the union over ranks is
    exactly the single-GPU workload (strong scaling)."""
    return slice(n * rank // world, n * (rank + 1) // world)


def c1():
    """Paper eq. (3): m1=m2=1, C1=C2=1012.5, x0=(1,0), v0=0 -> m, C, x0, v0 as [2]."""
    return (np.array([1.0, 1.0]), np.array([1012.5, 1012.5]),
            np.array([1.0, 0.0]), np.array([0.0, 0.0]))


def c2(B: int = C2_B):
    """[2][B]: m ~ U[0.5,2], C ~ U[500,2000], x0 ~ N(0,1), v0 = 0."""
    rng = _rng()
    m = rng.uniform(0.5, 2.0, (2, B))
    C = rng.uniform(500.0, 2000.0, (2, B))
    x0 = rng.standard_normal((2, B))
    return m, C, x0, np.zeros((2, B))


def c3(s: int = C3_S):
    """Single chain [s]: same distributions as C2."""
    rng = _rng()
    m = rng.uniform(0.5, 2.0, s)
    C = rng.uniform(500.0, 2000.0, s)
    x0 = rng.standard_normal(s)
    return m, C, x0, np.zeros(s)


def c4(B: int = C4_B, s: int = C4_S):
    """[B][s] batch of chains: same distributions as C2."""
    rng = _rng()
    m = rng.uniform(0.5, 2.0, (B, s))
    C = rng.uniform(500.0, 2000.0, (B, s))
    x0 = rng.standard_normal((B, s))
    return m, C, x0, np.zeros((B, s))


def c5(s: int = C5_S, N: int = C5_N):
    """Dense SPD system: M = diag(U[0.5,2]), K = Q diag(U[500,2000]) Q^T.

    Returns ``m [s]``, ``K [s][s]`` (symmetrised), ``X0 [s][N]``, ``V0 = 0``.
    """
    rng = _rng()
    m = rng.uniform(0.5, 2.0, s)
    c = rng.uniform(500.0, 2000.0, s)
    Q, R = np.linalg.qr(rng.standard_normal((s, s)))
    Q *= np.sign(np.diag(R))
    K = (Q * c) @ Q.T
    K = 0.5 * (K + K.T)
    X0 = rng.standard_normal((s, N))
    return m, K, X0, np.zeros((s, N))
