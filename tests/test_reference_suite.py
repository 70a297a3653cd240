"""The reference's own test suite, run against the B200 drop-in.

``python -m pytest -p paper_1702_02207_b200.dropin baseline/_ref/tests``:
the plugin rebinds ``oscbench``'s ``integrate``, ``rk4_step``,
``derivative`` and ``energy`` to the GPU path before the reference's tests
import them (paper_1702_02207_b200/dropin.py), so every trajectory, step,
derivative and energy those tests check -- including the bitwise
``run_parallel`` vs ``integrate`` contract (test_parallel.py:247-341), the
acceptance criteria (test_acceptance.py:100-158, 273-306) and the
``NonFiniteStateError`` cases (test_oscillator.py:119-123, 156-159) -- comes
from ``libosc_b200.so``.  The reference is the unmodified package installed
by scripts/install_reference.sh (baseline/_ref, with its tests/ and
configs/ beside it).
"""

import json
import os
import re
import subprocess
import sys

import pytest
from conftest import REF_INSTALL, ROOT

pytestmark = pytest.mark.gpu


def _run_reference_suite(tmp_path, *selection):
    tests = os.path.join(REF_INSTALL, "tests")
    if not os.path.isdir(tests):  # pragma: no cover
        pytest.skip("baseline/_ref/tests missing: run scripts/install_reference.sh")
    report = tmp_path / "dropin.json"
    ini = tmp_path / "pytest.ini"
    ini.write_text("[pytest]\n")
    env = dict(os.environ, PYTHONPATH=os.pathsep.join([REF_INSTALL, ROOT]),
               OSC_DROPIN_REPORT=str(report))
    cmd = [sys.executable, "-m", "pytest", "-c", str(ini), "--rootdir", REF_INSTALL,
           "-p", "no:cacheprovider", "-p", "paper_1702_02207_b200.dropin", "-q", "-rs",
           *(selection or (tests,))]
    res = subprocess.run(cmd, cwd=tmp_path, env=env, capture_output=True, text=True,
                         timeout=1500)
    out = res.stdout + res.stderr
    assert res.returncode == 0, out[-6000:]
    calls = json.loads(report.read_text())
    return out, calls


def test_reference_suite_passes_with_the_b200_drop_in(tmp_path):
    out, rep = _run_reference_suite(tmp_path)
    summary = out.strip().splitlines()[-1]
    assert re.search(r"\d+ passed", summary), summary
    assert "skipped" not in summary and "failed" not in summary, summary
    print(summary, rep["calls"])
    # every rebound function served the suite on the GPU
    for name in ("integrate", "rk4_step", "derivative", "energy"):
        assert rep["calls"][name] > 0, rep
    rebound = {tuple(r) for r in rep["rebound"]}
    for mod in ("oscbench", "oscbench.oscillator", "oscbench.harness"):
        assert (mod, "integrate") in rebound, rebound
