# Kernel change: full GPU parity suite, then C2 / C4 / C3 bench lines.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_gpu.log
for c in C2 C4 C3; do
  timeout 400 python bench.py --config $c --no-cpu --steps 3 > gpurun_out/bc_$c.json 2> gpurun_out/bc_$c.err; echo $c rc=$?
  python -c "import json; d=json.load(open('gpurun_out/bc_$c.json')); print('$c', '%.4g'%d['value'], round(d['ms_per_step'],2), round(d['roofline_fp64']['frac'],3), 'fma %.4g'%d['fma_mode']['value'], 'e2e %.4g'%d['e2e']['value'])"
done
