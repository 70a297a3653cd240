# K3 A/B: triple-buffered persistent tiles (default) vs the round-1 double buffer (pb2).
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_edge.py tests/test_gpu_sharded.py tests/test_gpu_validation.py -q -x > gpurun_out/pytest_c3ab.log 2>&1; echo pytest rc=$?
tail -2 gpurun_out/pytest_c3ab.log
for i in 1 2; do
timeout 600 python bench.py --config C3 --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/c3_pb3_$i.json 2>gpurun_out/c3_pb3.err; echo pb3 rc=$?
OSC_LIB=paper_1702_02207_b200/_variants/pb2/libosc_b200.so timeout 600 python bench.py --config C3 --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/c3_pb2_$i.json 2>gpurun_out/c3_pb2.err; echo pb2 rc=$?
done
python - <<'PY'
import json,glob
for f in sorted(glob.glob('gpurun_out/c3_pb*_*.json')):
    d=json.loads(open(f).read().strip().splitlines()[-1]); print(f, round(d['ms_per_step'],2), round(d['roofline']['frac'],4), d['roofline']['issue_frac'], d['clocks'])
PY
python scripts/prof_chain.py C3 96 > gpurun_out/plain_c3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:chain_tiles_persistent -s 1 -c 1 -o gpurun_out/prof_c3_pb3 python scripts/prof_chain.py C3 96 > gpurun_out/ncu_c3.log 2>&1; echo ncu rc=$?
