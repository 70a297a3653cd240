# One-system builds of K1 after a change: the K1 parity/edge tests, C1 latency, and the
# C2 slices of 4 and 8 GPUs (2^18, 2^17 systems) at the default launch shape.
timeout 900 python -m pytest tests/test_gpu_edge.py tests/test_gpu_parity.py tests/test_gpu_compare.py tests/test_gpu_hypothesis.py -x -q -m gpu 2>&1 | tail -2
timeout 300 python bench.py --config C1 --steps 3 --warmup 3 --no-cpu 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('C1 ms per 1e6 steps', round(d['ms_per_step'],3), 'e2e', d['e2e']['value'])"
python - <<'PY'
import torch, json
from paper_1702_02207_b200 import batched, workloads
full = workloads.c2()
for B in (1 << 18, 1 << 17, 1 << 16):
    m, C, x0, v0 = (torch.from_numpy(a[:, :B].copy()).cuda() for a in full)
    f = lambda: batched.integrate_batch2(m, C, x0, v0, 1e-4, 10000, check=False, validate=False)
    for _ in range(2): f()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(3): f()
    b.record(); torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 3
    print('B', B, 'ms', round(ms, 3), 'DOF-steps/s %.3e' % (2 * B * 10000 / ms * 1e3))
PY
