"""Throughput floors well below the measured numbers (profiles/r01): they
catch a silent fall back to the exact-division replay, a wrong launch shape
or a lost unroll -- regressions that keep every parity test green."""

import pytest

from paper_1702_02207_b200 import workloads

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_1702_02207_b200 import batched  # noqa: E402


def _rate(fn, dof_steps, reps=2):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return dof_steps * reps / (a.elapsed_time(b) * 1e-3)


def test_c2_throughput_floor():
    m, C, x0, v0 = (torch.from_numpy(a).cuda() for a in workloads.c2())
    p = workloads.PARAMS["C2"]
    rate = _rate(lambda: batched.integrate_batch2(m, C, x0, v0, p.dt, p.nsteps, check=False,
                                                  validate=False), m.numel() * p.nsteps)
    assert rate > 3.0e11, rate  # measured 3.81e11


def test_c4_throughput_floor():
    m, C, x0, v0 = (torch.from_numpy(a).cuda() for a in workloads.c4())
    p = workloads.PARAMS["C4"]
    rate = _rate(lambda: batched.integrate_chains(m, C, x0, v0, p.dt, p.nsteps, check=False,
                                                  validate=False), m.numel() * p.nsteps, reps=1)
    assert rate > 2.5e11, rate  # measured 3.14e11
