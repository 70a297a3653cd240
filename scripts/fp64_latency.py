"""Dependent-chain latency of DFMA / DADD / DMUL on this GPU (one thread,
clock64 cycles per op): the floor under C1's serial RK4 step."""
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1702_02207_b200 import _native  # noqa: E402

lib = _native.lib()
sink = torch.zeros(512, dtype=torch.float64, device="cuda")
out = {}
for mode, name in ((4, "dfma"), (5, "dadd"), (6, "dmul")):
    ops = ctypes.c_int64()
    for _ in range(2):  # warm-up, then measure
        assert lib.osc_bench_fp64(100_000, mode, ctypes.c_void_p(sink.data_ptr()),
                                  ctypes.byref(ops), None) == 0
        torch.cuda.synchronize()
    out[name + "_cycles_per_dependent_op"] = float(sink[0].item()) / ops.value
print(json.dumps(out))
