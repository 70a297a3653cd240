# C4 (whole chains): steps per launch (OSC_WHOLE_STEPS) -- launch boundaries
# vs the exact-replay granularity.
mkdir -p gpurun_out
for n in 512 1024 2000 2500 5000 10000; do
  OSC_WHOLE_STEPS=$n timeout 300 python bench.py --config C4 --steps 3 --warmup 3 --no-cpu --no-e2e --no-side > gpurun_out/c4ws.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/c4ws.json').read().strip().splitlines()[-1]); print('C4 whole steps/launch $n', round(d['ms_per_step'],2))"
done
