# C4 end to end vs the host pipeline's chunk count (OSC_HOST_CHUNKS).
set -x
for rep in 1 2; do
for n in 1 2 3 4 8; do
  OSC_HOST_CHUNKS=$n timeout 300 python bench.py --config C4 --steps 3 --warmup 3 --no-cpu --no-side > gpurun_out/c4ch_$n.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/c4ch_$n.json').read().strip().splitlines()[-1]);print('chunks=$n', round(d['ms_per_step'],3), '%.4g'%d['e2e']['value'], round(4.194304e10/d['e2e']['value']*1e3,3))"
done
done
