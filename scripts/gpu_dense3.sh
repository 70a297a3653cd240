set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_dense.py -x -q > gpurun_out/pytest_dense.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_dense.log
for cfg in "2,16,4" "2,32,3" "2,32,4"; do
OSC_DENSE=$cfg timeout 600 python bench.py --config C5 --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_C5_${cfg//,/_}.json 2>&1; echo $cfg rc=$?
done
