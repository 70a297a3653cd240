set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_multirank.py -x -q > gpurun_out/pytest_mr.log 2>&1; echo pytest rc=$?
tail -15 gpurun_out/pytest_mr.log
