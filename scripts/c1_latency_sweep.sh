# C1 latency: default latency build vs the compare build with compare off.
mkdir -p gpurun_out
for v in 0 1; do
  if [ $v = 1 ]; then export OSC_B2_LATCMP=1; fi
  timeout 300 python bench.py --config C1 --no-cpu --no-e2e --steps 5 > gpurun_out/c1v_$v.json 2> gpurun_out/c1v_$v.err
  python -c "import json; d=json.load(open('gpurun_out/c1v_$v.json')); print('variant $v', d['ms_per_step'], 'validation', d['validation']['ms_per_step'])"
done
