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


def collect(worker, args, nprocs):
    """Spawn nprocs ranks of worker(rank, *args, queue); return what rank 0
    puts on the queue.  Reads before joining (results larger than a pipe
    buffer would otherwise deadlock) and fails fast if a rank dies."""
    import queue as queue_mod

    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = mp.start_processes(worker, args=args + (q,), nprocs=nprocs, join=False,
                               start_method="spawn")
    while True:
        try:
            out = q.get(timeout=1.0)
            break
        except queue_mod.Empty:
            if procs.join(timeout=0):  # raises if a rank failed
                raise RuntimeError("ranks exited without a result")
    while not procs.join():
        pass
    return out
