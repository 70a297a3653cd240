# C3 tile shape x steps-per-launch sweep (persistent tiled kernel).
mkdir -p gpurun_out
for cfg in "8,256 32" "8,256 31" "8,256 30" "8,256 28" "8,128 16" "8,128 20" "8,128 24"; do
  set -- $cfg
  OSC_TILE=$1 timeout 300 python bench.py --config C3 --no-cpu --no-e2e --steps 3 --halo $2 \
    > gpurun_out/s3_$1_$2.json 2> gpurun_out/s3_$1_$2.err
  python -c "import json; d=json.load(open('gpurun_out/s3_$1_$2.json')); print('$1 T=$2', round(d['ms_per_step'],1), round(d['roofline_fp64']['frac'],3))"
done
