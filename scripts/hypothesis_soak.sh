# Large unseeded hypothesis run of the GPU property tests (bug hunt; not part
# of the suite).  HYPOTHESIS_SOAK scales max_examples in the test modules.
mkdir -p gpurun_out
export HYPOTHESIS_SOAK=${HYPOTHESIS_SOAK:-10}
timeout ${SOAK_TIMEOUT:-3000} python -m pytest tests/test_gpu_hypothesis.py tests/test_gpu_sharded.py tests/test_gpu_multirank.py -q -p no:cacheprovider \
  --hypothesis-show-statistics -k "random" > gpurun_out/soak.log 2>&1; echo soak rc=$?
grep -E "passing|passed|failed|Falsifying" gpurun_out/soak.log | head -30
