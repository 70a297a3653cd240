# K3 checked two-operation division: tests + C3 A/B (OSC_DIV2=0 = three operations).
set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py tests/test_gpu_sharded.py -q -x > gpurun_out/pytest_div2c.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_div2c.log
for i in 1 2; do
timeout 600 python bench.py --config C3 --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/c3_d2_$i.json 2>gpurun_out/c3_d2.err; echo d2 rc=$?
OSC_DIV2=0 timeout 600 python bench.py --config C3 --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/c3_d3_$i.json 2>gpurun_out/c3_d3.err; echo d3 rc=$?
done
python - <<'PY'
import json,glob
for f in sorted(glob.glob('gpurun_out/c3_d*_*.json')):
    d=json.loads(open(f).read().strip().splitlines()[-1]); print(f, round(d['ms_per_step'],2), round(d['roofline']['frac'],4), d['roofline'].get('issue_frac'), d['clocks'])
PY
