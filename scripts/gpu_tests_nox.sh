# GPU test pass without -x (every failure listed) + smoke.
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
timeout 1500 python -m pytest tests -q -m gpu -rs ${PYTEST_ARGS:-} > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
grep -E "FAILED|ERROR|passed|failed" gpurun_out/pytest_gpu.log | tail -30
