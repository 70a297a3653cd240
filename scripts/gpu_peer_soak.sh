# Multi-process fused-exchange tests + the >= 500-run soak (round 2).
set -x
mkdir -p gpurun_out
[ -n "$SKIP_TESTS" ] || { timeout 900 python -m pytest tests/test_gpu_multirank.py tests/test_gpu_sharded.py -q -x > gpurun_out/pytest_mr.log 2>&1; echo pytest rc=$?; }
tail -3 gpurun_out/pytest_mr.log
timeout 2400 python scripts/peer_soak.py --groups ${SOAK_GROUPS:-20} --runs ${SOAK_RUNS:-30} --budget 600 --out gpurun_out/peer_soak > gpurun_out/soak.log 2>&1; echo soak rc=$?
tail -3 gpurun_out/soak.log
