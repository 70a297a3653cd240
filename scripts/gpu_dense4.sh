set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_dense.py -x -q > gpurun_out/pytest_dense.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_dense.log
timeout 600 python bench.py --config C5 --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_C5_64x32.json 2>&1; echo rc=$?
python scripts/prof_dense.py 3 > gpurun_out/prof_dense_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:dense_rk4_gemm -s 2 -c 1 -o gpurun_out/prof_dense3 python scripts/prof_dense.py 3 > gpurun_out/ncu_dense.log 2>&1; echo ncu rc=$?
