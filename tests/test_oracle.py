"""Pin the CPU oracle to the reference's own outputs (tests/golden, made by
tests/golden/gen_golden.py running oscbench itself).  CPU only."""

import numpy as np
import pytest

import oracle
from conftest import bits, import_reference, reference_path
from paper_1702_02207_b200 import workloads
from paper_1702_02207_b200.oscillator import accumulated_times


def _cases(golden):
    for name in ("c1_paper", "canonical", "chain3", "chain64_stiff"):
        yield name, golden(name)


def test_c_oracle_matches_reference_trajectories(golden):
    for name, g in _cases(golden):
        xs, vs, x, v, fb = oracle.c_rk4_chains(g["m"][None], g["C"][None], g["x0"][None],
                                               g["v0"][None], float(g["dt"]), int(g["nsteps"]),
                                               int(g["stride"]))
        assert fb[0] == 0, name
        assert bits(xs[:, 0]) == bits(g["xs"]), name
        assert bits(vs[:, 0]) == bits(g["vs"]), name


def test_numpy_oracle_matches_reference_trajectories(golden):
    for name in ("canonical", "chain3", "chain64_stiff"):
        g = golden(name)
        xs, vs, fb = oracle.np_integrate(g["m"], g["C"], g["x0"], g["v0"], float(g["dt"]),
                                         int(g["nsteps"]), int(g["stride"]))
        assert fb == 0
        assert bits(xs) == bits(g["xs"]), name
        assert bits(vs) == bits(g["vs"]), name


def test_time_labels_match_reference(golden):
    for name in ("c1_paper", "canonical", "chain3", "chain64_stiff"):
        g = golden(name)
        t0 = float(g["t0"]) if "t0" in g else 0.0
        ts = accumulated_times(t0, float(g["dt"]), int(g["nsteps"]), int(g["stride"]))
        assert bits(ts) == bits(g["ts"]), name
    # C1 ends at the accumulated label, not 1e6 * 1e-4.
    assert golden("c1_paper")["ts"][-1] == 100.00000000219612


def test_c2_subset_batched_layout(golden):
    g = golden("c2_subset")
    xs, vs, x, v, fb = oracle.c_rk4_batch2(g["m"], g["C"], g["x0"], g["v0"], float(g["dt"]),
                                           int(g["nsteps"]), int(g["stride"]))
    assert not fb.any()
    assert bits(xs) == bits(g["xs"])
    assert bits(vs) == bits(g["vs"])


def test_c2_inputs_are_the_seeded_workload(golden):
    g = golden("c2_subset")
    m, C, x0, v0 = workloads.c2(B=1 << 12)
    # The first systems of a smaller draw differ (the draw is [2][B]); the
    # golden file stores the first 64 columns of the full-size draw.
    mf, Cf, x0f, _ = workloads.c2()
    assert bits(mf[:, :64]) == bits(g["m"]) and bits(x0f[:, :64]) == bits(g["x0"])
    assert m.shape == (2, 1 << 12)


def test_c4_subset_chains(golden):
    g = golden("c4_subset")
    xs, vs, x, v, fb = oracle.c_rk4_chains(g["m"], g["C"], g["x0"], g["v0"], float(g["dt"]),
                                           int(g["nsteps"]), int(g["stride"]))
    assert not fb.any()
    assert bits(xs) == bits(g["xs"])
    assert bits(vs) == bits(g["vs"])


def test_c4_full_horizon_chains(golden):
    """Two C4 chains over the full 10^4 steps of configs[3], sampled every
    1000 steps, as the reference computed them."""
    g = golden("c4_full_subset")
    xs, vs, x, v, fb = oracle.c_rk4_chains(g["m"], g["C"], g["x0"], g["v0"], float(g["dt"]),
                                           int(g["nsteps"]), int(g["stride"]))
    assert not fb.any()
    assert bits(xs) == bits(g["xs"]) and bits(vs) == bits(g["vs"])


@pytest.mark.parametrize("where", ["wall", "free", "mid"])
def test_c3_light_cone_windows(golden, where):
    g = golden(f"c3_window_{where}")
    n = int(g["nsteps"])
    _, _, x, v, fb = oracle.c_rk4_chains(g["m"][None], g["C"][None], g["x0"][None],
                                         np.zeros_like(g["x0"])[None], float(g["dt"]), n, n,
                                         sample=False)
    a, lo = int(g["a"]), int(g["lo"])
    w = int(g["b"]) - a
    assert bits(x[0, a - lo:a - lo + w]) == bits(g["x"])
    assert bits(v[0, a - lo:a - lo + w]) == bits(g["v"])


def test_mt_chain_is_bit_identical_to_sequential(golden):
    g = golden("chain64_stiff")
    x, v, fb = oracle.c_rk4_chain_mt(g["m"], g["C"], g["x0"], g["v0"], float(g["dt"]),
                                     int(g["nsteps"]), nthreads=4)
    assert fb == 0
    assert bits(x) == bits(g["xs"][-1]) and bits(v) == bits(g["vs"][-1])


def test_divergence_steps_match_reference(golden):
    e = golden("edge")
    for tag, dt in (("div1e9", 1e9), ("div1e3", 1e3), ("div2e-2", 2e-2)):
        _, _, _, _, fb = oracle.c_rk4_chains([[0.002, 0.002]], [[20250.0, 20250.0]],
                                             [[2.0, -3.0]], [[0.0, 0.0]], dt, 1000, 1)
        assert fb[0] == int(e[f"{tag}_first_bad"]), tag
        _, _, fbn = oracle.np_integrate([0.002, 0.002], [20250.0, 20250.0], [2.0, -3.0],
                                        [0.0, 0.0], dt, 1000, 1)
        assert fbn == int(e[f"{tag}_first_bad"]), tag


def test_signed_zero_equilibrium(golden):
    e = golden("edge")
    xs, vs, _, _, fb = oracle.c_rk4_chains([[0.002, 0.002]], [[20250.0, 20250.0]],
                                           [[0.0, -0.0]], [[-0.0, 0.0]], 0.25, 3, 1)
    assert bits(xs[:, 0]) == bits(e["eq_xs"]) and bits(vs[:, 0]) == bits(e["eq_vs"])


def test_derivative_and_energy_known_answers(golden):
    e = golden("edge")
    d = oracle.c_derivative([0.002, 0.002], [20250.0, 20250.0], [2.0, -3.0])[0]
    assert bits(d) == bits(e["canon_dvel"])
    assert tuple(d) == (-70_875_000.0, 50_625_000.0)
    E = oracle.c_energy([0.002, 0.002], [20250.0, 20250.0], [2.0, -3.0], [0.0, 0.0])[0]
    assert E == e["canon_energy"] == 293_625.0
    d3 = oracle.c_derivative([0.5, 1.0, 2.0], [3.0, 4.0, 5.0], [0.3, -0.2, 0.7])[0]
    assert bits(d3) == bits(e["chain3_dvel"])
    E3 = oracle.c_energy([0.5, 1.0, 2.0], [3.0, 4.0, 5.0], [0.3, -0.2, 0.7], [0.1, 0.0, -0.4])
    assert bits(E3) == bits(e["chain3_energy"])


def test_c1_against_analytic_modes(golden):
    g = golden("c1_paper")
    sol = oracle.analytic_solution(1.0, 1012.5, (1.0, 0.0), (0.0, 0.0))
    assert sol[0] == pytest.approx(51.48552625359159, abs=1e-12)
    assert sol[1] == pytest.approx(19.665721100196947, abs=1e-12)
    err, rmse, at = oracle.compare(g["ts"], g["xs"], sol)
    assert err < 1.1e-7 and rmse <= err  # 1.069e-7 m, rmse 3.016e-8


def test_dense_restatement_tracks_analytic():
    m, K, X0, V0 = workloads.c5(s=48, N=4)
    A = K / m[:, None]
    X, V = oracle.dense_rk4(A, X0, V0, 1e-4, 200)
    Xa = oracle.dense_analytic(m, K, X0, 200 * 1e-4)
    assert np.max(np.abs(X - Xa)) <= 1e-8 * np.max(np.abs(X0))


# --------------------------------------------------------------------------
# property-based parity against the reference itself (build container only:
# the reference package is not on the GPU box)
# --------------------------------------------------------------------------


from hypothesis import given, settings, strategies as st  # noqa: E402

_REF = reference_path()


@pytest.mark.skipif(_REF is None, reason="reference package not present")
@settings(max_examples=40, deadline=None, derandomize=True)
@given(s=st.integers(1, 9), nsteps=st.integers(1, 60), stride=st.integers(1, 7),
       seed=st.integers(0, 2**32 - 1), dt=st.sampled_from([1e-4, 1e-3, 5e-3, 2e-2]))
def test_c_oracle_equals_reference_on_random_chains(s, nsteps, stride, seed, dt):
    oscbench = import_reference()

    rng = np.random.default_rng(seed)
    m = rng.uniform(0.3, 3.0, s)
    C = rng.uniform(100.0, 3000.0, s)
    x0 = rng.standard_normal(s) * rng.choice([1e-3, 1.0, 1e3])
    v0 = rng.standard_normal(s)
    x0[rng.random(s) < 0.2] = 0.0
    try:
        traj = oscbench.integrate(oscbench.build_chain(m, C), oscbench.PhaseState(x0, v0),
                                  dt, nsteps, stride)
        ref_bad = 0
    except oscbench.NonFiniteStateError as exc:
        ref_bad = exc.step
    xs, vs, _, _, fb = oracle.c_rk4_chains(m[None], C[None], x0[None], v0[None], dt, nsteps,
                                           stride)
    assert fb[0] == ref_bad
    if not ref_bad:
        assert bits(xs[:, 0]) == bits(np.array([p.positions for p in traj.samples]))
        assert bits(vs[:, 0]) == bits(np.array([p.velocities for p in traj.samples]))


# --------------------------------------------------------------------------
# modal analytic solution and compare (modal.py:98-162), pinned to
# tests/golden/modal.npz (the reference's own analytic_solution / compare)
# --------------------------------------------------------------------------

def test_modal_restatement_matches_reference(golden):
    g = golden("modal")
    for i in range(len(g["m"])):
        sol = oracle.analytic_solution(g["m"][i], g["C"][i], g["x0"][i], g["v0"][i])
        assert bits(np.array(sol)) == bits(g["sol"][i]), i
        gen = oracle.analytic_general(g["m"][i], g["m"][i], g["C"][i], g["C"][i], g["x0"][i],
                                      g["v0"][i])
        assert bits(np.array(gen)) == bits(g["sol"][i]), i


def test_compare_restatement_matches_reference(golden):
    g = golden("modal")
    rep = g["report"]
    assert bits(np.array(oracle.compare_seq(g["c1_ts"], g["c1_xs"], g["sol"][0]))) == bits(rep[0])
    assert bits(np.array(oracle.compare_seq(g["canon_ts"], g["canon_xs"],
                                            g["sol"][1]))) == bits(rep[1])
    for b in range(g["rand_xs"].shape[-1]):
        got = oracle.compare_seq(g["rand_ts"], g["rand_xs"][:, :, b], g["sol"][2 + b])
        assert bits(np.array(got)) == bits(rep[2 + b]), b


def test_general_modal_solution_is_the_exact_solution():
    """Unequal parameters (outside modal.py): each mode solves the pencil,
    and the fit reproduces the initial positions and velocities."""
    rng = np.random.default_rng(3)
    for _ in range(200):
        m0, m1 = rng.uniform(0.5, 2.0, 2)
        C0, C1 = rng.uniform(500.0, 2000.0, 2)
        x0, v0 = rng.standard_normal(2), rng.standard_normal(2) * 10
        w1, w2, r1, r2, a1c, a1s, a2c, a2s = oracle.analytic_general(m0, m1, C0, C1, x0, v0)
        K = np.array([[C0 + C1, -C1], [-C1, C1]])
        M = np.diag([m0, m1])
        lam = np.sort(np.linalg.eigvals(np.linalg.solve(M, K)).real)[::-1]
        assert np.allclose([w1 * w1, w2 * w2], lam, rtol=1e-12)
        for w, r in ((w1, r1), (w2, r2)):
            res = (K - w * w * M) @ np.array([1.0, r])
            assert np.abs(res).max() <= 1e-9 * np.abs(K).max() * (1 + abs(r))
        x1a, x2a = oracle.eval_analytic((w1, w2, r1, r2, a1c, a1s, a2c, a2s), [0.0])
        assert np.allclose([x1a[0], x2a[0]], x0, atol=1e-13)
        vel0 = np.array([w1 * a1s + w2 * a2s, r1 * w1 * a1s + r2 * w2 * a2s])
        assert np.allclose(vel0, v0, atol=1e-11)
