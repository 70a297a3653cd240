# Host-pointer pipeline check: validation/host-form tests + the default bench line (e2e).
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_validation.py tests/test_gpu_c_abi.py tests/test_gpu_parity.py tests/test_gpu_hypothesis.py -q -x > gpurun_out/pytest_e2e.log 2>&1; echo pytest rc=$?
tail -2 gpurun_out/pytest_e2e.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_e2e.json 2> gpurun_out/bench_e2e.err; echo bench rc=$?
python -c "import json;d=json.loads(open('gpurun_out/bench_e2e.json').read().strip().splitlines()[-1]);print(d['value'], d['e2e']['value'], d['ms_per_step'], d['roofline']['frac'], d['clocks'])"
