# C3 tile shapes with the current K3 (one-test division, bulk stores).
mkdir -p gpurun_out
for cfg in "8,256 31" "8,128 16" "8,128 24" "8,128 32"; do
  set -- $cfg
  OSC_TILE=$1 timeout 600 python bench.py --config C3 --halo $2 --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/c3t.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/c3t.json')); print('C3 tile $1 T=$2', round(d['ms_per_step'],2))"
done
