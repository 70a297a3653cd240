# Chain launch-shape sweep (C4 whole-chain, C3 persistent tiles).
set -x
mkdir -p gpurun_out
for w in "8,128" "4,256"; do
  OSC_WHOLE=$w timeout 300 python bench.py --config C4 --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/sw_C4_${w/,/x}.json 2>&1; echo C4 $w rc=$?
done
for cfg in "8,256 32" "4,512 32" "4,256 32" "4,512 48"; do
  set -- $cfg
  OSC_TILE=$1 timeout 300 python bench.py --config C3 --halo $2 --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/sw_C3_${1/,/x}_T$2.json 2>&1; echo C3 $cfg rc=$?
done
OSC_TILE=4,512 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "tiled or c3 or persistent" > gpurun_out/pytest_k4.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pytest_k4.log
