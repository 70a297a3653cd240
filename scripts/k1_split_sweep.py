"""K1 launch shapes for the per-rank slices of C2 at N = 1, 2, 4, 8 GPUs
(2^20 / N systems): the strong split shrinks the batch, and a shape that is
right for 2^20 systems can leave a partly filled last wave at 2^17.  Times
one integrate_batch2 of the first B systems for each OSC_B2 shape (set per
subprocess: the launcher reads it per call) and prints a JSON table."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import sys, json, torch
sys.path.insert(0, %r)
from paper_1702_02207_b200 import batched, workloads
B = int(sys.argv[1])
m, C, x0, v0 = (torch.from_numpy(a[:, :B].copy()).cuda() for a in workloads.c2())
f = lambda: batched.integrate_batch2(m, C, x0, v0, 1e-4, 10000, check=False, validate=False)
for _ in range(2): f()
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(3): f()
b.record(); torch.cuda.synchronize()
print(json.dumps({"ms": a.elapsed_time(b) / 3}))
''' % ROOT

out = {}
for n in (1, 2, 4, 8):
    B = (1 << 20) // n
    for shape in ("default", "1,256", "2,256", "2,128", "2,64", "1,128", "1,64"):
        env = dict(os.environ)
        if shape != "default":
            env["OSC_B2"] = shape
        r = subprocess.run([sys.executable, "-c", CHILD, str(B)], env=env, capture_output=True,
                           text=True)
        try:
            ms = json.loads(r.stdout.strip().splitlines()[-1])["ms"]
        except Exception:  # noqa: BLE001
            ms = None
        out[f"B={B} {shape}"] = ms
        print(f"B={B} shape={shape} ms={ms} DOFsteps/s={2 * B * 1e4 / (ms * 1e-3) if ms else None:.4g}",
              flush=True)
print(json.dumps(out))
