"""The gpu scenario wired into the reference harness.

Runs in the build container where the reference package is importable (it is
absent on the GPU box, so this is a CPU test): the GPU integrate is replaced
by the reference's own integrate to check the glue -- dispatch by scenario
name, the determinism verdict, the analytic/energy checks and the CSV report
all come from the unchanged reference harness."""

import os
import sys

import pytest

REF = "/root/reference/pkg/src"
if not os.path.isdir(REF):  # pragma: no cover - GPU box
    pytest.skip("reference package not present", allow_module_level=True)
sys.path.insert(0, REF)

import oscbench  # noqa: E402
import oscbench.harness  # noqa: E402

from paper_1702_02207_b200 import harness as gpu_harness  # noqa: E402

INI = """
[system]
masses = 0.002, 0.002
springs = 20250, 20250
[initial]
x0 = 2, -3
v0 = 0, 0
[run]
dt = 1e-6
nsteps = 2000
stride = 100
warmup = 100
[scenario seq]
[scenario gpu]
"""


def test_gpu_scenario_runs_through_reference_harness(tmp_path):
    calls = []

    def fake_integrate(system, state0, dt, nsteps, stride):
        calls.append((dt, nsteps, stride))
        return oscbench.integrate(system, state0, dt, nsteps, stride)

    uninstall = gpu_harness.install(oscbench, integrate=fake_integrate,
                                    timer=lambda fn: (fn(), 1e-3))
    try:
        config = oscbench.parse_config(INI)
        runner = oscbench.BenchRunner(config)
        results = runner.run_all()
    finally:
        uninstall()
    assert oscbench.harness.run_parallel is not None
    names = [r.name for r in results]
    assert names == ["seq", "gpu"]
    gpu = results[1]
    assert calls == [(1e-6, 2000, 100)]
    assert gpu.determinism is True  # bitwise against the cached reference
    assert gpu.max_abs_err is not None and gpu.max_abs_err < 1e-6
    assert gpu.energy_drift_rel < 1e-6
    assert gpu.pooled.count == 1900 and abs(gpu.pooled.mean - 5e-7) < 1e-15
    summary, samples = oscbench.write_csv(results, str(tmp_path / "run"))
    lines = open(summary).read().splitlines()
    assert lines[2].startswith("gpu,1,") and ",pass," in lines[2]


def test_uninstall_restores_parallel_engine():
    original = oscbench.harness.run_parallel
    uninstall = gpu_harness.install(oscbench, integrate=oscbench.integrate,
                                    timer=lambda fn: (fn(), 1.0))
    assert oscbench.harness.run_parallel is not original
    uninstall()
    assert oscbench.harness.run_parallel is original


def test_reference_rebinding_routes_the_cli_integrate_command(tmp_path, capsys):
    """install(reference=True): the CLI's integrate command (cli.py:119-135,
    via BenchRunner.reference) calls the injected integrate; uninstall
    restores every rebound name."""
    import oscbench.cli

    calls = []
    ref_integrate = oscbench.harness.integrate

    def fake_integrate(system, state0, dt, nsteps, stride=1):
        calls.append(nsteps)
        return ref_integrate(system, state0, dt, nsteps, stride)

    originals = (oscbench.harness.integrate, oscbench.integrate, oscbench.oscillator.integrate)
    ini = tmp_path / "run.ini"
    ini.write_text(INI)
    uninstall = gpu_harness.install(oscbench, integrate=fake_integrate, reference=True,
                                    timer=lambda fn: (fn(), 1e-3))
    try:
        rc = oscbench.cli.main(["integrate", "--config", str(ini)])
    finally:
        uninstall()
    assert rc == 0 and calls == [2000]
    assert "max_abs_err_m=" in capsys.readouterr().out
    assert (oscbench.harness.integrate, oscbench.integrate,
            oscbench.oscillator.integrate) == originals
