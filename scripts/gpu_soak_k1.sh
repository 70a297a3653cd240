# Random soak of K1 after the state-range tests: test_batch2_random at HYPOTHESIS_SOAK x the
# suite's examples, for the default launch shapes (one-system builds at these sizes) and with
# the two-systems build forced.
mkdir -p gpurun_out
export HYPOTHESIS_SOAK=${HYPOTHESIS_SOAK:-10}
for shape in default 2,256 1,32; do
  if [ $shape = default ]; then unset OSC_B2; else export OSC_B2=$shape; fi
  timeout ${SOAK_TIMEOUT:-1500} python -m pytest tests/test_gpu_hypothesis.py -q -p no:cacheprovider \
    --hypothesis-show-statistics -k "batch2_random" > gpurun_out/soak_k1_$shape.log 2>&1; echo soak $shape rc=$?
  grep -E "passing examples|passed|failed|Falsifying|events" -A0 gpurun_out/soak_k1_$shape.log | head -8
  grep -E "^\s+\* [0-9.]+%" gpurun_out/soak_k1_$shape.log | head -12
done
