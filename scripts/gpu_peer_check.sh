set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
timeout 900 python -m pytest tests/test_gpu_multirank.py tests/test_gpu_sharded.py tests/test_gpu_validation.py tests/test_gpu_fullsize.py -q -x -rs > gpurun_out/pytest_mr.log 2>&1; echo pytest rc=$?
tail -5 gpurun_out/pytest_mr.log
timeout 600 python scripts/peer_soak.py --groups 4 --runs 10 --budget 200 --out gpurun_out/peer_soak_small > gpurun_out/soak_small.log 2>&1; echo soak rc=$?
tail -3 gpurun_out/soak_small.log
