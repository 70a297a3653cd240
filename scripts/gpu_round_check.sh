# Full GPU test suite + bench lines of C2, C3, C4 (quick), for a commit check.
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_gpu.log
for c in C3 C4 C2; do timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu > gpurun_out/rc_$c.json 2> gpurun_out/rc_$c.err; echo bench $c rc=$?; done
python - <<'PY'
import json
for c in ("C3","C4","C2"):
    try:
        d=json.loads(open(f'gpurun_out/rc_{c}.json').read().strip().splitlines()[-1])
        print(c, round(d['ms_per_step'],2), d['value'], d['roofline']['frac'], d['roofline'].get('issue_frac'), d.get('e2e',{}).get('value'), d['clocks']['sm_mhz'], d['clocks']['reasons'])
    except Exception as e: print(c, 'ERR', e)
PY
