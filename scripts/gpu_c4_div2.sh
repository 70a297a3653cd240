set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_hypothesis.py tests/test_gpu_fullsize.py -q -x -k "chain or c4 or div or tile or tiled" > gpurun_out/pytest_c4.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_c4.log
for i in 1 2; do
timeout 600 python bench.py --config C4 --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/c4d2_$i.json 2>gpurun_out/c4d2.err; echo c4 rc=$?
OSC_DIV2=0 timeout 600 python bench.py --config C4 --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/c4d3_$i.json 2>gpurun_out/c4d3.err; echo c4div3 rc=$?
done
python - <<'PY'
import json,glob
for f in sorted(glob.glob('gpurun_out/c4d*_*.json')):
    d=json.loads(open(f).read().strip().splitlines()[-1]); print(f, round(d['ms_per_step'],2), d['roofline']['frac'], d['roofline'].get('issue_frac'), d['clocks']['sm_mhz'], d['clocks']['reasons'])
PY
