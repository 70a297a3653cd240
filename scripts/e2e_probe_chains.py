"""C4's end-to-end overhead: device integrate_chains (resident) vs the
host-pointer call, at the full 10^4 steps and at 1 step (the fixed cost:
copies, parameter check, table, allocations), for the default host plan
(three chunks: small first/last) and the OSC_HOST_CHUNKS / OSC_HOST_EDGE
alternatives."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1702_02207_b200 import _native, batched, workloads  # noqa: E402

m, C, x0, v0 = workloads.c4()
B, s = x0.shape
dev = [torch.from_numpy(a).cuda() for a in (m, C, x0, v0)]
lib = _native.lib()
pin = [torch.from_numpy(np.ascontiguousarray(a)).pin_memory() for a in (m, C, x0, v0)]
x, v = pin[2].clone().pin_memory(), pin[3].clone().pin_memory()
fb = torch.empty(B, dtype=torch.int64).pin_memory()
PLANS = [("default", {}), ("chunks=1", {"OSC_HOST_CHUNKS": "1"}),
         ("chunks=8", {"OSC_HOST_CHUNKS": "8"}), ("edge=8", {"OSC_HOST_EDGE": "8"}),
         ("edge=32", {"OSC_HOST_EDGE": "32"})]
ref = None
for nsteps in (10000, 1):
    f = lambda: batched.integrate_chains(*dev, 1e-4, nsteps, check=False)  # noqa: E731
    r = f()
    torch.cuda.synchronize()
    if nsteps == 10000:
        ref = (r.x.cpu().numpy().tobytes(), r.v.cpu().numpy().tobytes())
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(3):
        f()
    b.record()
    torch.cuda.synchronize()
    print("nsteps=%d device %.2f ms" % (nsteps, a.elapsed_time(b) / 3))
    for name, env in PLANS:
        for k in ("OSC_HOST_CHUNKS", "OSC_HOST_EDGE"):
            os.environ.pop(k, None)
        os.environ.update(env)
        ts = []
        for i in range(4):
            x.copy_(pin[2])
            v.copy_(pin[3])
            torch.cuda.synchronize()
            t = time.perf_counter()
            rc = lib.osc_rk4_chains_host(pin[0].data_ptr(), pin[1].data_ptr(), x.data_ptr(),
                                         v.data_ptr(), B, s, 1e-4, nsteps, nsteps, None, None,
                                         fb.data_ptr())
            ts.append((time.perf_counter() - t) * 1e3)
            assert rc == 0, rc
        same = ""
        if nsteps == 10000:
            same = " bytes-equal" if (x.numpy().tobytes(), v.numpy().tobytes()) == ref else " DIFFER"
        print("nsteps=%d host %s: %s ms%s" % (nsteps, name, " ".join("%.2f" % t for t in ts[1:]),
                                              same))
