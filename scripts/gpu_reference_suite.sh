# The reference's own test suite against the B200 drop-in, evidence for profiles/r02.
set -x
mkdir -p gpurun_out
printf '[pytest]\n' > /tmp/ref_pytest.ini
cd /tmp && OSC_DROPIN_REPORT=/tmp/dropin_calls.json PYTHONPATH=$GRAFT_REPO_ROOT/baseline/_ref:$GRAFT_REPO_ROOT \
  timeout 1500 python -m pytest -c /tmp/ref_pytest.ini --rootdir $GRAFT_REPO_ROOT/baseline/_ref \
  -p no:cacheprovider -p paper_1702_02207_b200.dropin $GRAFT_REPO_ROOT/baseline/_ref/tests -v -rA \
  > $GRAFT_REPO_ROOT/gpurun_out/reference_suite_gpu.txt 2>&1; echo rc=$?
cd $GRAFT_REPO_ROOT
cp /tmp/dropin_calls.json gpurun_out/dropin_calls.json
tail -3 gpurun_out/reference_suite_gpu.txt; cat gpurun_out/dropin_calls.json | head -20
