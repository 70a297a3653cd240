set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm --format=csv > gpurun_out/smi.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests/test_reference_suite.py tests/test_harness_gpu_scenario.py -q -s -rs > gpurun_out/refsuite.log 2>&1
echo rc=$?
tail -30 gpurun_out/refsuite.log
