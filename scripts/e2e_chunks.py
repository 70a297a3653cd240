"""C2 end to end through osc_rk4_batch2_host (pinned buffers) for several
chunk counts (OSC_HOST_CHUNKS; read per call)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1702_02207_b200 import _native, workloads  # noqa: E402

lib = _native.lib()
m, C, x0, v0 = (torch.from_numpy(np.ascontiguousarray(a)).pin_memory() for a in workloads.c2())
x, v = torch.empty_like(x0).pin_memory(), torch.empty_like(v0).pin_memory()
B = x0.shape[1]
fb = torch.empty(B, dtype=torch.int64).pin_memory()
for n in sys.argv[1:]:
    os.environ["OSC_HOST_CHUNKS"] = n
    ts = []
    for i in range(5):
        x.copy_(x0)
        v.copy_(v0)
        torch.cuda.synchronize()
        t = time.perf_counter()
        rc = lib.osc_rk4_batch2_host(m.data_ptr(), C.data_ptr(), x.data_ptr(), v.data_ptr(), B,
                                     1e-4, 10_000, 10_000, None, None, fb.data_ptr())
        ts.append(time.perf_counter() - t)
        assert rc == 0
    print(f"chunks={n}: {min(ts[2:])*1e3:.2f} ms (median {sorted(ts[2:])[1]*1e3:.2f})", flush=True)
