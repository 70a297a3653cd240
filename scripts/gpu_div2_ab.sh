# Two-operation division: GPU tests, then C2/C1 with it on and off (A/B).
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_hypothesis.py tests/test_gpu_edge.py tests/test_gpu_compare.py -x -q -m gpu > gpurun_out/pytest_div2.log 2>&1; echo pytest rc=$?
tail -5 gpurun_out/pytest_div2.log
for c in C2 C1; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu > gpurun_out/ab_${c}_on.json 2> gpurun_out/ab_${c}_on.err; echo on $c rc=$?
  OSC_DIV2=0 timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/ab_${c}_off.json 2> gpurun_out/ab_${c}_off.err; echo off $c rc=$?
done
python - <<'PY'
import json
for c in ("C2","C1"):
    for k in ("on","off"):
        try:
            d=json.load(open(f"gpurun_out/ab_{c}_{k}.json"))
            print(c,k,d["value"],d["ms_per_step"],d["roofline_fp64"]["frac"],d["roofline_fp64"]["dp_inst_per_dof_step"])
        except Exception as e: print(c,k,"ERR",e)
PY
