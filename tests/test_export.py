"""Trajectory export: the CSV is byte-identical to the
reference's export_trajectory (harness.py:607-621); npz is lossless."""

import os
import sys

import numpy as np
import pytest

import paper_1702_02207_b200 as osc
from conftest import import_reference
from paper_1702_02207_b200 import export


def _traj(golden, name):
    g = golden(name)
    t0 = float(g["t0"]) if "t0" in g else 0.0
    samples = [osc.PhaseState(g["xs"][j], g["vs"][j], g["ts"][j]) for j in range(len(g["ts"]))]
    assert samples[0].time == t0
    return osc.Trajectory(tuple(samples), float(g["dt"]), int(g["stride"]))


@pytest.mark.parametrize("name", ["canonical", "chain3", "chain64_stiff"])
def test_csv_matches_reference_exporter(golden, tmp_path, name):
    traj = _traj(golden, name)
    ours = tmp_path / "ours.csv"
    export.export_trajectory(traj, str(ours))
    oscbench = import_reference()
    if oscbench is None:  # pragma: no cover - run scripts/install_reference.sh
        pytest.skip("reference package not present")
    from oscbench.harness import export_trajectory as ref_export

    theirs = tmp_path / "theirs.csv"
    rtraj = oscbench.Trajectory(tuple(oscbench.PhaseState(s.positions, s.velocities, s.time)
                                      for s in traj.samples), traj.dt, traj.stride)
    ref_export(rtraj, str(theirs))
    assert ours.read_bytes() == theirs.read_bytes()


def test_npz_is_lossless(golden, tmp_path):
    traj = _traj(golden, "chain64_stiff")
    path = str(tmp_path / "t.npz")
    export.export_npz(traj, path)
    with np.load(path) as z:
        g = golden("chain64_stiff")
        assert z["positions"].tobytes() == g["xs"].tobytes()
        assert z["velocities"].tobytes() == g["vs"].tobytes()
        assert z["times"].tobytes() == g["ts"].tobytes()
