# Chain kernels: parity tests + C3 (checked two-op default / OSC_DIV2=0) + C4 bench lines.
set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py tests/test_gpu_sharded.py tests/test_gpu_hypothesis.py -q -x > gpurun_out/pytest_chain.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_chain.log
for i in 1 2; do
timeout 600 python bench.py --config C3 --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/cab_c3_$i.json 2>gpurun_out/cab_c3.err; echo c3 rc=$?
OSC_DIV2=0 timeout 600 python bench.py --config C3 --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/cab_c3div3_$i.json 2>gpurun_out/cab_c3div3.err; echo c3div3 rc=$?
timeout 600 python bench.py --config C4 --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/cab_c4_$i.json 2>gpurun_out/cab_c4.err; echo c4 rc=$?
done
python - <<'PY'
import json,glob
for f in sorted(glob.glob('gpurun_out/cab_*.json')):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1]); print(f, round(d['ms_per_step'],2), d['clocks']['sm_mhz'], d['clocks']['reasons'])
    except Exception as e: print(f, 'ERR', e)
PY
