# Two-operation division (K1: C2, C1): GPU tests, then each config with it on and off (A/B).
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -5 gpurun_out/pytest_gpu.log
for c in ${CONFIGS:-C2 C1}; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/ab_${c}_on.json 2> gpurun_out/ab_${c}_on.err; echo on $c rc=$?
  OSC_DIV2=0 timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/ab_${c}_off.json 2> gpurun_out/ab_${c}_off.err; echo off $c rc=$?
done
python - <<'PY'
import json, os
for c in os.environ.get("CONFIGS", "C2 C1").split():
    for k in ("on","off"):
        try:
            d=json.load(open(f"gpurun_out/ab_{c}_{k}.json"))
            print(c,k,d["value"],d["ms_per_step"],d["roofline_fp64"]["frac"],d["roofline_fp64"]["dp_inst_per_dof_step"])
        except Exception as e: print(c,k,"ERR",e)
PY
