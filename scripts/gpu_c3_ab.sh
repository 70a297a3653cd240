# C3 A/B: skewed persistent tiles (injection period 4/8/16) vs the strided kernel.
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py tests/test_gpu_sharded.py tests/test_gpu_hypothesis.py -x -q -m gpu > gpurun_out/pt_c3.log 2>&1; echo pytest rc=$?; tail -1 gpurun_out/pt_c3.log
for v in "1 4" "1 8" "1 16" "0 4"; do
  set -- $v
  OSC_SKEW=$1 OSC_SKEW_INJ=$2 timeout 300 python bench.py --config C3 --no-cpu --no-e2e --steps 3 > gpurun_out/c3ab_$1_$2.json 2> gpurun_out/c3ab_$1_$2.err
  python -c "import json; d=json.load(open('gpurun_out/c3ab_$1_$2.json')); print('OSC_SKEW=$1 inj=$2', round(d['ms_per_step'],1), round(d['roofline_fp64']['frac'],3))"
done
