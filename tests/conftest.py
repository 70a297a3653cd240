import os
import sys

import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")

# The unmodified reference package: the install under baseline/_ref
# (scripts/install_reference.sh; travels to the GPU box) or, in the build
# container only, the read-only source tree.
REF_INSTALL = os.path.join(ROOT, "baseline", "_ref")
REF_SOURCE = "/root/reference/pkg/src"


def reference_path():
    """Directory to put on sys.path to import ``oscbench``, or None."""
    for cand in (REF_INSTALL, REF_SOURCE):
        if os.path.isfile(os.path.join(cand, "oscbench", "__init__.py")):
            return cand
    return None


def import_reference():
    """Import the reference package ``oscbench`` (or None when absent)."""
    path = reference_path()
    if path is None:
        return None
    if path not in sys.path:
        sys.path.insert(0, path)
    import oscbench

    return oscbench


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libosc_b200.so")


@pytest.fixture(scope="session")
def golden():
    import numpy as np

    cache = {}

    def load(name):
        if name not in cache:
            with np.load(os.path.join(GOLDEN, name + ".npz")) as z:
                cache[name] = {k: z[k] for k in z.files}
        return cache[name]

    return load


def bits(a):
    """Exact byte image (like the reference's conftest.trajectory_bits)."""
    import numpy as np

    return np.ascontiguousarray(np.asarray(a, dtype="<f8")).tobytes()


def collect(worker, args, nprocs, timeout=240.0):
    """Spawn nprocs ranks of worker(rank, *args, queue); return what rank 0
    puts on the queue.  Reads before joining (results larger than a pipe
    buffer would otherwise deadlock) and fails fast if a rank dies.  Bounded:
    after `timeout` seconds, or on any error (pytest-timeout included), the
    ranks are terminated, so a stuck rank cannot keep the test session alive."""
    import queue as queue_mod
    import time

    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = mp.start_processes(worker, args=args + (q,), nprocs=nprocs, join=False,
                               start_method="spawn")
    deadline = time.monotonic() + timeout
    try:
        while True:
            try:
                out = q.get(timeout=1.0)
                break
            except queue_mod.Empty:
                if procs.join(timeout=0):  # raises if a rank failed
                    raise RuntimeError("ranks exited without a result")
                if time.monotonic() > deadline:
                    raise TimeoutError(f"{nprocs} ranks gave no result in {timeout:.0f} s")
        while not procs.join(timeout=max(1.0, deadline - time.monotonic())):
            if time.monotonic() > deadline:
                raise TimeoutError(f"{nprocs} ranks did not exit in {timeout:.0f} s")
        return out
    finally:
        for p in procs.processes:
            if p.is_alive():
                p.terminate()
        for p in procs.processes:
            p.join(5.0)
            if p.is_alive():
                p.kill()
