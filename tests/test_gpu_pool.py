"""The library's scratch comes from its own memory pool: the device's default
pool (the host application's cudaMallocAsync) keeps its release threshold
(round 1 raised it process-wide)."""

import ctypes
import ctypes.util
import glob

import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_1702_02207_b200 import batched, workloads  # noqa: E402


def _cudart():
    for cand in ["libcudart.so.12", ctypes.util.find_library("cudart"),
                 *glob.glob("/usr/local/cuda/lib64/libcudart.so*")]:
        if cand:
            try:
                return ctypes.CDLL(cand)
            except OSError:
                continue
    pytest.skip("libcudart not found")


def _default_pool_threshold(rt, dev=0):
    pool = ctypes.c_void_p()
    assert rt.cudaDeviceGetDefaultMemPool(ctypes.byref(pool), dev) == 0
    val = ctypes.c_uint64(12345)
    attr_release_threshold = 4  # cudaMemPoolAttrReleaseThreshold
    assert rt.cudaMemPoolGetAttribute(pool, attr_release_threshold, ctypes.byref(val)) == 0
    return val.value


def test_default_pool_untouched_by_library_calls():
    rt = _cudart()
    before = _default_pool_threshold(rt)
    m, C, x0, v0 = workloads.c4(B=8, s=4000)
    batched.integrate_chains(m, C, x0, v0, 1e-4, 64)        # scratch (ping-pong buffers)
    mm, CC, xx, vv = workloads.c2(B=4096)
    batched.integrate_batch2(mm, CC, xx, vv, 1e-4, 100)     # scratch (division classes)
    torch.cuda.synchronize()
    assert _default_pool_threshold(rt) == before

