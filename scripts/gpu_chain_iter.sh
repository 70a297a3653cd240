# Chain-kernel iteration: parity subset, C3/C4 bench lines, ncu of the K3 tile kernel.
set -x
mkdir -p gpurun_out
TAG=${TAG:-iter}
timeout 900 python -m pytest tests/test_gpu_edge.py tests/test_gpu_sharded.py tests/test_gpu_validation.py tests/test_gpu_parity.py -q -x > gpurun_out/pytest_$TAG.log 2>&1; echo pytest rc=$?
tail -2 gpurun_out/pytest_$TAG.log
for c in C3 C4; do
timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/${c}_$TAG.json 2>gpurun_out/${c}_$TAG.err; echo $c rc=$?
done
python - <<'PY'
import json,glob,os
tag=os.environ.get('TAG','iter')
for c in ('C3','C4'):
    f=f'gpurun_out/{c}_{tag}.json'
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1]); print(c, round(d['ms_per_step'],2), round(d['roofline']['frac'],4), round(d['roofline']['issue_frac'],4), d['clocks'])
    except Exception as e: print(c, 'ERR', e)
PY
if [ -z "$NO_NCU" ]; then
python scripts/prof_chain.py C3 96 > gpurun_out/plain_c3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:chain_tiles_persistent -s 1 -c 1 -o gpurun_out/prof_c3_$TAG python scripts/prof_chain.py C3 96 > gpurun_out/ncu_c3.log 2>&1; echo ncu rc=$?
fi
