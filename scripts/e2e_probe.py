"""Where C2's end-to-end time goes: the device step (resident inputs), the
same batch cut into n chunks on n streams (resident), and the host-pointer
call with n chunks (OSC_HOST_CHUNKS).  Prints ms per full C2 run."""
import ctypes
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1702_02207_b200 import _native, batched, workloads  # noqa: E402

m, C, x0, v0 = workloads.c2()
dev = [torch.from_numpy(a).cuda() for a in (m, C, x0, v0)]


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def chunked(n):
    B = m.shape[1]
    parts = [(B * c // n, B * (c + 1) // n) for c in range(n)]
    sl = [[t[:, lo:hi].contiguous() for t in dev] for lo, hi in parts]
    streams = [torch.cuda.Stream() for _ in range(n)]

    def run():
        cur = torch.cuda.current_stream()
        for s, p in zip(streams, sl):
            s.wait_stream(cur)
            with torch.cuda.stream(s):
                batched.integrate_batch2(*p, 1e-4, 10000, check=False, validate=False)
        for s in streams:
            cur.wait_stream(s)
    return run


print("device, one launch: %.2f ms" % timed(
    lambda: batched.integrate_batch2(*dev, 1e-4, 10000, check=False, validate=False)))
for n in (2, 4):
    print("device, %d chunks on %d streams: %.2f ms" % (n, n, timed(chunked(n))))
lib = _native.lib()
pin = [torch.from_numpy(np.ascontiguousarray(a)).pin_memory() for a in (m, C, x0, v0)]
x, v = pin[2].clone().pin_memory(), pin[3].clone().pin_memory()
fb = torch.empty(m.shape[1], dtype=torch.int64).pin_memory()
for n in ("1", "2", "4"):
    os.environ["OSC_HOST_CHUNKS"] = n
    ts = []
    for i in range(4):
        x.copy_(pin[2])
        v.copy_(pin[3])
        torch.cuda.synchronize()
        t = time.perf_counter()
        rc = lib.osc_rk4_batch2_host(pin[0].data_ptr(), pin[1].data_ptr(), x.data_ptr(),
                                     v.data_ptr(), m.shape[1], 1e-4, 10000, 10000, None, None,
                                     fb.data_ptr())
        ts.append((time.perf_counter() - t) * 1e3)
    print("host call, OSC_HOST_CHUNKS=%s: %s ms" % (n, " ".join("%.2f" % t for t in ts[1:])))
