"""The gpu scenario wired into the reference harness.

The reference package comes from baseline/_ref (scripts/install_reference.sh,
which travels to the GPU box) or the build container's source tree.  The CPU
tests inject the reference's own integrate to check the glue -- dispatch by
scenario name, the determinism verdict, the analytic/energy checks and the
CSV report all come from the unchanged reference harness; the ``gpu`` tests
run the same scenarios with the real B200 integrate and nothing injected."""

import pytest
from conftest import import_reference

oscbench = import_reference()
if oscbench is None:  # pragma: no cover - run scripts/install_reference.sh
    pytest.skip("reference package not present", allow_module_level=True)

import oscbench.cli  # noqa: E402
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


@pytest.mark.gpu
def test_gpu_scenario_on_the_b200_through_reference_harness(tmp_path):
    """[scenario gpu] with the real GPU integrate: the reference harness's
    bitwise determinism verdict compares the B200 trajectory with its own
    cached sequential integrate (harness.py:486-502) and passes."""
    uninstall = gpu_harness.install(oscbench)
    try:
        runner = oscbench.BenchRunner(oscbench.parse_config(INI))
        results = runner.run_all()
    finally:
        uninstall()
    assert [r.name for r in results] == ["seq", "gpu"]
    gpu = results[1]
    assert gpu.determinism is True
    assert gpu.max_abs_err is not None and gpu.max_abs_err < 1e-6
    assert gpu.energy_drift_rel < 1e-6
    assert gpu.pooled.count == 1900 and gpu.pooled.mean > 0.0
    summary, _ = oscbench.write_csv(results, str(tmp_path / "run"))
    lines = open(summary).read().splitlines()
    assert lines[2].startswith("gpu,1,") and ",pass," in lines[2]


@pytest.mark.gpu
def test_cli_integrate_command_on_the_b200(tmp_path, capsys):
    """install(reference=True): the reference CLI's integrate command
    (cli.py:119-135) runs on the B200 and prints the reference's report."""
    ini = tmp_path / "run.ini"
    ini.write_text(INI)
    ref = oscbench.harness.integrate
    uninstall = gpu_harness.install(oscbench, reference=True)
    try:
        assert oscbench.harness.integrate is not ref
        rc = oscbench.cli.main(["integrate", "--config", str(ini)])
    finally:
        uninstall()
    assert rc == 0
    assert "max_abs_err_m=" in capsys.readouterr().out
    assert oscbench.harness.integrate is ref
