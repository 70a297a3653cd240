set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_validation.py tests/test_gpu_parity.py tests/test_gpu_c_abi.py tests/test_gpu_edge.py tests/test_harness_gpu_scenario.py -q -x > gpurun_out/pytest_v.log 2>&1; echo pytest rc=$?
tail -2 gpurun_out/pytest_v.log
python scripts/dropin_latency.py > gpurun_out/dropin_latency.json 2>&1; cat gpurun_out/dropin_latency.json
bash scripts/gpu_reference_suite.sh
