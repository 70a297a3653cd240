"""Full BASELINE configurations checked exactly where the oracle can follow:
C3 (one 2^24-cell chain, all 10^4 steps, default plan) byte-equal at three
light-cone windows -- cells [a, b) after n steps depend only on cells
[a - 2n, b + 2n) -- and C5 (s = 4096, 1024 trajectories, 1000
steps) against the generalized-eigen analytic solution (1e-8
relative)."""

import os

import numpy as np
import pytest

import oracle
from conftest import bits
from paper_1702_02207_b200 import workloads

pytestmark = [pytest.mark.gpu, pytest.mark.timeout(900)]

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_1702_02207_b200 import batched  # noqa: E402


def test_c3_full_run_light_cone_windows():
    m, C, x0, v0 = workloads.c3()
    p = workloads.PARAMS["C3"]
    s, n = m.shape[0], p.nsteps
    res = batched.integrate_chains(m, C, x0, v0, p.dt, n)
    x, v = res.x[0].cpu().numpy(), res.v[0].cpu().numpy()
    w = 256
    for a in (0, s // 2 - w // 2, s - w):
        lo, hi = max(0, a - 2 * n), min(s, a + w + 2 * n)
        xo, vo, fb = oracle.c_rk4_chain_mt(m[lo:hi], C[lo:hi], x0[lo:hi], v0[lo:hi], p.dt, n,
                                           nthreads=os.cpu_count() or 1)
        assert fb == 0
        assert bits(x[a:a + w]) == bits(xo[a - lo:a - lo + w]), a
        assert bits(v[a:a + w]) == bits(vo[a - lo:a - lo + w]), a


def test_c5_full_run_against_analytic():
    m, K, X0, V0 = workloads.c5()
    p = workloads.PARAMS["C5"]
    A = batched.rowscale(torch.from_numpy(K).cuda(), torch.from_numpy(m).cuda())
    res = batched.integrate_dense(A, X0, V0, p.dt, p.nsteps)
    Xa = oracle.dense_analytic(m, K, X0, p.nsteps * p.dt)
    # relative to the solution itself (not to the initial amplitude)
    err = np.max(np.abs(res.x.cpu().numpy() - Xa)) / np.max(np.abs(Xa))
    assert err <= 1e-8, err


def test_c5_full_size_64_steps_against_restatement():
    """configs[4] at full size (s=4096, 1024 trajectories) for 64 steps
    against the numpy restatement (oracle.dense_rk4, CPU BLAS): GEMM
    summation order differs, so 1e-10 relative, positions and
    velocities, each relative to its own magnitude."""
    m, K, X0, V0 = workloads.c5()
    p = workloads.PARAMS["C5"]
    A = K / m[:, None]
    n = 64
    res = batched.integrate_dense(A, X0, V0, p.dt, n)
    Xo, Vo = oracle.dense_rk4(A, X0, V0, p.dt, n)
    ex = np.max(np.abs(res.x.cpu().numpy() - Xo)) / np.max(np.abs(Xo))
    ev = np.max(np.abs(res.v.cpu().numpy() - Vo)) / np.max(np.abs(Vo))
    assert ex <= 1e-10 and ev <= 1e-10, (ex, ev)


@pytest.mark.parametrize("transport", ["nccl", "peer"])
def test_c3_full_run_eight_shards_equal_one_gpu(transport):
    """The full C3 chain in 8 shards (LocalShardGroup: same kernels, layouts
    and exchange logic as the multi-GPU driver, all on this device), all 10^4
    steps, byte-equal to the single-GPU run over every cell."""
    from paper_1702_02207_b200 import sharded

    m, C, x0, v0 = workloads.c3()
    p = workloads.PARAMS["C3"]
    ref = batched.integrate_chains(m, C, x0, v0, p.dt, p.nsteps)
    grp = sharded.LocalShardGroup(m, C, x0, v0, p.dt, 8, transport=transport)
    assert grp.run(p.nsteps) == 0
    x, v = grp.gather()
    assert torch.equal(x.view(torch.int64), ref.x[0].view(torch.int64))
    assert torch.equal(v.view(torch.int64), ref.v[0].view(torch.int64))
