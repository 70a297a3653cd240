"""Small driver for profiling the dense GEMM (C5 shape, a few RK4 steps)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1702_02207_b200 import batched, workloads  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
m, K, X0, V0 = workloads.c5()
A = batched.rowscale(K, m)
res = batched.integrate_dense(A, X0, V0, 1e-4, steps, check=False)
torch.cuda.synchronize()
print("ok", float(res.x[0, 0]))
