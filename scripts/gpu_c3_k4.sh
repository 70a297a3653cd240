# C3 with 4-cell threads (16 warps per SM) vs the default 8-cell build, both
# with the three-operation division (OSC_DIV2=0: the 4-cell builds have no
# two-operation form yet).
mkdir -p gpurun_out
for cfg in "8,256 31" "4,512 31" "4,512 24" "4,512 40" "4,256 16" "4,256 24"; do
  set -- $cfg
  OSC_DIV2=0 OSC_TILE=$1 timeout 600 python bench.py --config C3 --halo $2 --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/c3k4.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/c3k4.json')); print('C3 div3 tile $1 T=$2', round(d['ms_per_step'],2))"
done
OSC_TILE=8,256 timeout 600 python bench.py --config C3 --halo 31 --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/c3k4.json 2>/dev/null
python -c "import json; d=json.load(open('gpurun_out/c3k4.json')); print('C3 default div2 8,256 T=31', round(d['ms_per_step'],2))"
