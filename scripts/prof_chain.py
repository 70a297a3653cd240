"""Small driver for profiling the chain kernels: C3 tiled (one chain of 2^24
cells) or C4 whole-chain (4096 x 1024), a few launches."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1702_02207_b200 import batched, workloads  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 64
if cfg == "C3":
    m, C, x0, v0 = workloads.c3()
    res = batched.integrate_chains(m, C, x0, v0, 1e-4, steps, check=False)
else:
    m, C, x0, v0 = workloads.c4()
    res = batched.integrate_chains(m, C, x0, v0, 1e-4, steps, check=False)
torch.cuda.synchronize()
print("ok", float(res.x[0, 0]))
