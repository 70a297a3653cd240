# C3 steps per launch (T) with the round-2 K3: rounds x (T + transition) vs halo share.
mkdir -p gpurun_out
for T in 24 28 30 31 32 36 40 48; do
  timeout 300 python bench.py --config C3 --halo $T --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/c3_T$T.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/c3_T$T.json').read().strip().splitlines()[-1]);print('T=$T', round(d['ms_per_step'],2), round(d['roofline']['issue_frac'],4), d['clocks']['sm_mhz'])"
done
