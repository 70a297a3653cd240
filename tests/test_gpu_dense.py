"""K5 dense path vs the restatement oracle (numpy, fp64 BLAS) and the
eigen-analytic solution.  Tolerances: relative max-abs <= 1e-10
against the restatement (GEMM summation order differs), <= 1e-8 against the
analytic solution."""

import numpy as np
import pytest

import oracle
from paper_1702_02207_b200 import workloads

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_1702_02207_b200 import batched  # noqa: E402

REL_RESTATEMENT = 1e-10
REL_ANALYTIC = 1e-8


def _relerr(a, b):
    return float(np.max(np.abs(a - b)) / np.max(np.abs(b)))


def test_rowscale_is_exact_division():
    m, K, _, _ = workloads.c5(s=300, N=4)
    A = batched.rowscale(K, m).cpu().numpy()
    assert A.tobytes() == (K / m[:, None]).tobytes()


@pytest.mark.parametrize("s,N,nsteps", [(128, 32, 50), (48, 7, 40), (300, 70, 30),
                                        (512, 256, 20)])
def test_dense_matches_restatement(s, N, nsteps):
    m, K, X0, V0 = workloads.c5(s=s, N=N)
    V0 = np.random.default_rng(s).standard_normal((s, N))  # exercise the velocity terms
    A = K / m[:, None]
    res = batched.integrate_dense(A, X0, V0, 1e-4, nsteps)
    Xo, Vo = oracle.dense_rk4(A, X0, V0, 1e-4, nsteps)
    assert _relerr(res.x.cpu().numpy(), Xo) <= REL_RESTATEMENT
    assert _relerr(res.v.cpu().numpy(), Vo) <= REL_RESTATEMENT


def test_dense_matches_analytic_and_is_deterministic():
    s, N, n = 256, 64, 300
    m, K, X0, V0 = workloads.c5(s=s, N=N)
    A = batched.rowscale(K, m)
    r1 = batched.integrate_dense(A, X0, V0, 1e-4, n)
    r2 = batched.integrate_dense(A, X0, V0, 1e-4, n)
    assert r1.x.cpu().numpy().tobytes() == r2.x.cpu().numpy().tobytes()
    Xa = oracle.dense_analytic(m, K, X0, n * 1e-4)
    assert _relerr(r1.x.cpu().numpy(), Xa) <= REL_ANALYTIC


def test_dense_c5_shape_short_run():
    """configs[4] at full size (s=4096, N=1024), 3 steps vs the restatement."""
    m, K, X0, V0 = workloads.c5()
    A = K / m[:, None]
    res = batched.integrate_dense(A, X0, V0, 1e-4, 3)
    Xo, Vo = oracle.dense_rk4(A, X0, V0, 1e-4, 3)
    assert _relerr(res.x.cpu().numpy(), Xo) <= REL_RESTATEMENT
    assert _relerr(res.v.cpu().numpy(), Vo) <= REL_RESTATEMENT


def test_dense_divergence_flag():
    m, K, X0, V0 = workloads.c5(s=128, N=32)
    res = batched.integrate_dense(K / m[:, None], X0, V0, 10.0, 200, check=False)
    assert int(res.first_bad[0]) > 0
