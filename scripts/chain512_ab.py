"""Whole chains of 512 cells (K = 4 whole-chain kernel), one library per
process (OSC_LIB): ms per 2048-step run."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1702_02207_b200 import batched, workloads  # noqa: E402

m, C, x0, v0 = (torch.as_tensor(a).cuda() for a in workloads.c4(B=8192, s=512))
batched.integrate_chains(m, C, x0, v0, 1e-4, 512)
torch.cuda.synchronize()
ts = []
for _ in range(3):
    t = time.perf_counter()
    batched.integrate_chains(m, C, x0, v0, 1e-4, 2048)
    torch.cuda.synchronize()
    ts.append(time.perf_counter() - t)
print(os.environ.get("OSC_LIB", "current"), f"{min(ts) * 1e3:.2f} ms")
