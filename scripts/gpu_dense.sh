# Dense path: tests, then bench C5 (short), then a full ncu capture of one GEMM.
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_dense.py -x -q > gpurun_out/pytest_dense.log 2>&1; echo pytest rc=$?
tail -15 gpurun_out/pytest_dense.log
timeout 900 python bench.py --config C5 --steps 3 --warmup 3 > gpurun_out/bench_C5.json 2> gpurun_out/bench_C5.err; echo bench rc=$?
tail -c 2500 gpurun_out/bench_C5.json; tail -5 gpurun_out/bench_C5.err
