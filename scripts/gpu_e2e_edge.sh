# C2 end-to-end through the host-pointer ABI vs the small edge chunks of the
# host pipeline (OSC_HOST_EDGE=k: first/last chunk B/k; 0 = equal chunks).
set -x
for rep in 1 2; do
for ed in ${EDGES:-0 16 32}; do
  OSC_HOST_EDGE=$ed timeout 300 python bench.py --config C2 --steps 5 --warmup 3 --no-cpu --no-side > gpurun_out/e2e_$ed.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/e2e_$ed.json').read().strip().splitlines()[-1]);print('edge=$ed', round(d['ms_per_step'],3), '%.4g'%d['e2e']['value'], round(2.097152e10/d['e2e']['value']*1e3,3))"
done
done
