# C2 launch-shape sweep + tests (round 1).
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_gpu.log
for sh in "1,256" "1,128" "2,128" "2,256" "4,128" "4,64" "2,64"; do
  OSC_B2=$sh timeout 300 python bench.py --config C2 --steps 5 --warmup 3 --no-cpu > gpurun_out/sweep_C2_${sh/,/x}.json 2>&1; echo sweep C2 $sh rc=$?
done
timeout 600 python bench.py --config C4 --steps 5 --warmup 3 --no-cpu > gpurun_out/bench_C4.json 2>&1; echo C4 rc=$?
timeout 600 python bench.py --config C3 --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_C3.json 2>&1; echo C3 rc=$?
