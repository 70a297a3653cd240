"""Generate the golden fixtures by running the REFERENCE package itself.

Run in the build container (the reference does not exist on the GPU box):

    PYTHONPATH=/root/reference/pkg/src:/root/repo python tests/golden/gen_golden.py [modal|c4full]

Every fixture is the output of ``oscbench.integrate`` / ``oscbench.energy`` /
``oscbench.derivative`` (oscillator.py:184-276) on the inputs stored beside it,
with the accumulated time labels and the exact first-divergence step.  The
committed ``.npz`` files are what the oracle and the GPU path are pinned to.
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

import oscbench
from oscbench import NonFiniteStateError, PhaseState, build_chain, integrate

sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..", "..")))
from paper_1702_02207_b200 import workloads  # noqa: E402  (seeded inputs only)

OUT = os.path.dirname(os.path.abspath(__file__))


def run(masses, springs, x0, v0, dt, nsteps, stride, t0=0.0):
    """One reference integration -> dict of arrays (samples, times, first_bad)."""
    system = build_chain(list(masses), list(springs))
    state = PhaseState(tuple(x0), tuple(v0), t0)
    try:
        traj = integrate(system, state, dt, nsteps, stride)
    except NonFiniteStateError as exc:
        return {"first_bad": np.int64(exc.step)}
    xs = np.array([s.positions for s in traj.samples])
    vs = np.array([s.velocities for s in traj.samples])
    ts = np.array(traj.times())
    return {"xs": xs, "vs": vs, "ts": ts, "first_bad": np.int64(0)}


def save(name, **arrays):
    path = os.path.join(OUT, name + ".npz")
    np.savez_compressed(path, **arrays)
    print(f"wrote {path} ({os.path.getsize(path)} B)")


def main():
    t_start = time.time()

    # C1 -- BASELINE configs[0]: the paper's equal-parameter system, full run.
    m, C, x0, v0 = workloads.c1()
    p = workloads.PARAMS["C1"]
    r = run(m, C, x0, v0, p.dt, p.nsteps, p.stride)
    save("c1_paper", m=m, C=C, x0=x0, v0=v0, dt=p.dt, nsteps=p.nsteps, stride=p.stride, **r)

    # Canonical config of the reference tests (conftest.py:8-11, canonical.ini).
    r = run([0.002, 0.002], [20250.0, 20250.0], (2.0, -3.0), (0.0, 0.0), 1e-6, 10_000, 100)
    save("canonical", m=np.array([0.002, 0.002]), C=np.array([20250.0, 20250.0]),
         x0=np.array([2.0, -3.0]), v0=np.zeros(2), dt=1e-6, nsteps=10_000, stride=100, **r)

    # C2 subset: the first 64 seeded systems of configs[1], full 10^4 steps.
    m, C, x0, v0 = workloads.c2()
    nb = 64
    p = workloads.PARAMS["C2"]
    xs, vs = [], []
    for b in range(nb):
        r = run(m[:, b], C[:, b], x0[:, b], v0[:, b], p.dt, p.nsteps, 1000)
        xs.append(r["xs"])
        vs.append(r["vs"])
    save("c2_subset", m=m[:, :nb], C=C[:, :nb], x0=x0[:, :nb], v0=v0[:, :nb], dt=p.dt,
         nsteps=p.nsteps, stride=1000, xs=np.stack(xs, -1), vs=np.stack(vs, -1),
         ts=r["ts"])

    # Three-mass chain with uneven ownership (test_parallel.py:283-289).
    r = run([0.5, 1.0, 2.0], [3.0, 4.0, 5.0], (0.3, -0.2, 0.7), (0.1, 0.0, -0.4),
            1e-3, 100, 10)
    save("chain3", m=np.array([0.5, 1.0, 2.0]), C=np.array([3.0, 4.0, 5.0]),
         x0=np.array([0.3, -0.2, 0.7]), v0=np.array([0.1, 0.0, -0.4]), dt=1e-3,
         nsteps=100, stride=10, **r)

    # C4 subset: the first 2 seeded chains of configs[3] (s=1024), 1000 steps.
    m, C, x0, v0 = workloads.c4(B=2)
    xs, vs = [], []
    for b in range(2):
        r = run(m[b], C[b], x0[b], v0[b], 1e-4, 1000, 100)
        xs.append(r["xs"])
        vs.append(r["vs"])
    save("c4_subset", m=m, C=C, x0=x0, v0=v0, dt=1e-4, nsteps=1000, stride=100,
         xs=np.stack(xs, 1), vs=np.stack(vs, 1), ts=r["ts"])

    # C3 light-cone windows: wall end, free end and one interior window of the
    # 2^24-cell seeded chain after n steps (dependency radius 2 cells/step).
    m, C, x0, v0 = workloads.c3()
    s = m.shape[0]
    n, w = 100, 256
    wins = {"wall": (0, w), "free": (s - w, s), "mid": (s // 2 - w // 2, s // 2 + w // 2)}
    for name, (a, b) in wins.items():
        lo, hi = max(0, a - 2 * n), min(s, b + 2 * n)
        r = run(m[lo:hi], C[lo:hi], x0[lo:hi], v0[lo:hi], 1e-4, n, n)
        save(f"c3_window_{name}", a=a, b=b, lo=lo, hi=hi, nsteps=n, dt=1e-4,
             x=r["xs"][-1][a - lo:b - lo], v=r["vs"][-1][a - lo:b - lo],
             m=m[lo:hi], C=C[lo:hi], x0=x0[lo:hi])

    # Random 64-cell chain, stiff dt (omega*dt ~ 0.5): rounding-sensitive case,
    # with negative zeros and exact zeros in the initial state.
    rng = np.random.default_rng(7)
    m = rng.uniform(0.5, 2.0, 64)
    C = rng.uniform(500.0, 2000.0, 64)
    x0 = rng.standard_normal(64)
    v0 = rng.standard_normal(64)
    x0[[3, 17]] = -0.0
    x0[[5, 40]] = 0.0
    v0[[9, 63]] = -0.0
    r = run(m, C, x0, v0, 5e-3, 400, 40, t0=0.25)
    save("chain64_stiff", m=m, C=C, x0=x0, v0=v0, dt=5e-3, nsteps=400, stride=40,
         t0=0.25, **r)

    # Edge cases of the reference tests.
    edge = {}
    # s = 1 oscillator vs cos (test_oscillator.py:103-106), 10 steps dt=0.1.
    r = run([1.0], [1.0], (1.0,), (0.0,), 0.1, 10, 1)
    edge.update(s1_xs=r["xs"], s1_vs=r["vs"], s1_ts=r["ts"])
    # equilibrium keeps +-0 and accumulates time (test_oscillator.py:96-101).
    r = run([0.002, 0.002], [20250.0, 20250.0], (0.0, -0.0), (-0.0, 0.0), 0.25, 3, 1, t0=1.5)
    edge.update(eq_xs=r["xs"], eq_vs=r["vs"], eq_ts=r["ts"])
    # divergence step tagging (test_oscillator.py:119-123, 156-159).
    for tag, dt in (("div1e9", 1e9), ("div1e3", 1e3), ("div2e-2", 2e-2)):
        r = run([0.002, 0.002], [20250.0, 20250.0], (2.0, -3.0), (0.0, 0.0), dt, 1000, 1)
        edge[f"{tag}_first_bad"] = r["first_bad"]
    # derivative / energy known answers (test_oscillator.py:58-64, 172-174).
    sys2 = build_chain([0.002, 0.002], [20250.0, 20250.0])
    st = PhaseState((2.0, -3.0), (0.0, 0.0))
    edge["canon_dvel"] = np.array(oscbench.derivative(sys2, st).dvel)
    edge["canon_energy"] = np.float64(oscbench.energy(sys2, st))
    sys3 = build_chain([0.5, 1.0, 2.0], [3.0, 4.0, 5.0])
    st3 = PhaseState((0.3, -0.2, 0.7), (0.1, 0.0, -0.4))
    edge["chain3_dvel"] = np.array(oscbench.derivative(sys3, st3).dvel)
    edge["chain3_energy"] = np.float64(oscbench.energy(sys3, st3))
    save("edge", **edge)

    modal_fixture()
    print(f"done in {time.time() - t_start:.1f} s")


def modal_fixture():
    """modal.analytic_solution + integrate + modal.compare (modal.py:98-162)
    on equal-parameter systems: the paper's C1 system, the canonical test
    system and seeded random ones (m, C, x0, v0 all varied, v0 != 0)."""
    from oscbench import modal

    rng = np.random.default_rng(1702)
    cases = [(1.0, 1012.5, (1.0, 0.0), (0.0, 0.0)),
             (0.002, 20250.0, (2.0, -3.0), (0.0, 0.0))]
    for _ in range(14):
        cases.append((float(rng.uniform(0.5, 2.0)), float(rng.uniform(500.0, 2000.0)),
                      tuple(float(a) for a in rng.standard_normal(2)),
                      tuple(float(a) for a in rng.standard_normal(2) * 10.0)))
    # (dt, nsteps, stride) per case: C1 a shortened paper run, canonical the
    # reference tests' config, the random ones 2000 steps at omega*dt <= 0.1
    runs = [(1e-4, 100_000, 100), (1e-6, 10_000, 100)] + [(1e-3, 2000, 10)] * 14
    sol, rep, xs_all, ts_all = [], [], [], []
    for (m, c, x0, v0), (dt, n, stride) in zip(cases, runs):
        a = modal.analytic_solution(m, c, x0, v0)
        sol.append([a.omega1, a.omega2, a.r1, a.r2, a.a1c, a.a1s, a.a2c, a.a2s])
        traj = integrate(build_chain([m, m], [c, c]), PhaseState(x0, v0), dt, n, stride)
        r = modal.compare(traj, a)
        rep.append([r.max_abs_error, r.rmse, r.at_time])
        xs_all.append(np.array([s.positions for s in traj.samples]))
        ts_all.append(np.array(traj.times()))
    # the random cases share one shape: stack them as one [nsamp][2][B] batch
    save("modal", m=np.array([c[0] for c in cases]), C=np.array([c[1] for c in cases]),
         x0=np.array([c[2] for c in cases]), v0=np.array([c[3] for c in cases]),
         run=np.array(runs, dtype=np.float64), sol=np.array(sol), report=np.array(rep),
         c1_xs=xs_all[0], c1_ts=ts_all[0], canon_xs=xs_all[1], canon_ts=ts_all[1],
         rand_xs=np.stack(xs_all[2:], -1), rand_ts=ts_all[2])


def c4_full_fixture():
    """Two seeded C4 chains (s = 1024) over the FULL 10^4-step horizon of
    configs[3], sampled every 1000 steps (the reference takes ~40 s/chain):
    chains 0 and 1 of the full seeded C4 draw."""
    m, C, x0, v0 = (a[:2].copy() for a in workloads.c4())
    p = workloads.PARAMS["C4"]
    xs, vs = [], []
    for b in range(2):
        r = run(m[b], C[b], x0[b], v0[b], p.dt, p.nsteps, 1000)
        xs.append(r["xs"])
        vs.append(r["vs"])
    save("c4_full_subset", m=m, C=C, x0=x0, v0=v0, dt=p.dt, nsteps=p.nsteps, stride=1000,
         xs=np.stack(xs, 1), vs=np.stack(vs, 1), ts=r["ts"])


if __name__ == "__main__":
    if sys.argv[1:] == ["modal"]:
        modal_fixture()
    elif sys.argv[1:] == ["c4full"]:
        c4_full_fixture()
    else:
        main()
