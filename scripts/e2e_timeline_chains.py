"""Timeline of one C4 host-pointer call (torch.profiler / CUPTI sees the
library's kernels and copies): where the end-to-end overhead goes."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_1702_02207_b200 import _native, workloads  # noqa: E402

m, C, x0, v0 = workloads.c4()
B, s = x0.shape
lib = _native.lib()
pin = [torch.from_numpy(np.ascontiguousarray(a)).pin_memory() for a in (m, C, x0, v0)]
x, v = pin[2].clone().pin_memory(), pin[3].clone().pin_memory()
fb = torch.empty(B, dtype=torch.int64).pin_memory()
nsteps = int(sys.argv[1]) if len(sys.argv) > 1 else 10000


def call():
    x.copy_(pin[2])
    v.copy_(pin[3])
    torch.cuda.synchronize()
    t = time.perf_counter()
    rc = lib.osc_rk4_chains_host(pin[0].data_ptr(), pin[1].data_ptr(), x.data_ptr(),
                                 v.data_ptr(), B, s, 1e-4, nsteps, nsteps, None, None,
                                 fb.data_ptr())
    assert rc == 0
    return (time.perf_counter() - t) * 1e3


call()
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    wall = call()
evs = [e for e in prof.events() if e.device_type.name == "CUDA"]
evs.sort(key=lambda e: e.time_range.start)
t0 = min(e.time_range.start for e in evs)
print("wall %.2f ms" % wall)
for e in evs:
    print("%9.3f %9.3f ms  %-60s" % ((e.time_range.start - t0) / 1e3,
                                     (e.time_range.end - e.time_range.start) / 1e3, e.name[:60]))
