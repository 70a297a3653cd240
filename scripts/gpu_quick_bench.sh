# GPU suite + bench lines of the given configs (CONFIGS, default C4 C3 C2).
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -1 gpurun_out/pytest_gpu.log
for c in ${CONFIGS:-C4 C3 C2}; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/q_$c.json 2> gpurun_out/q_$c.err
  python -c "import json; d=json.load(open('gpurun_out/q_$c.json')); print('$c', round(d['ms_per_step'],2), round(d['roofline_fp64']['frac'] or 0,3), d['clocks']['reasons'])"
done
