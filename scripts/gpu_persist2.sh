set -x
mkdir -p gpurun_out
for cfg in "8,128 32" "8,256 32" "8,256 48" "8,256 64" "8,128 48"; do
  set -- $cfg
  OSC_TILE=$1 timeout 300 python bench.py --config C3 --halo $2 --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/p2_C3_${1/,/x}_T$2.json 2>&1; echo C3 $cfg rc=$?
done
OSC_TILE=8,256 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "tiled or c3" > gpurun_out/pytest_p2.log 2>&1; echo pytest rc=$?
tail -2 gpurun_out/pytest_p2.log
