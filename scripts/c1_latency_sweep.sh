# C1 latency vs the K1 latency-path build, plus the C2 headline for the same build.
mkdir -p gpurun_out
for lb in 0 32; do
  OSC_B2_LB=$lb OSC_B2=1,32 timeout 300 python bench.py --config C1 --no-cpu --no-e2e --steps 5 \
    > gpurun_out/c1lat_$lb.json 2> gpurun_out/c1lat_$lb.err
  python -c "import json; d=json.load(open('gpurun_out/c1lat_$lb.json')); print('C1 LB=$lb', d['ms_per_step'], 'ms/1e6 steps; validation', d['validation']['ms_per_step'])"
done
timeout 300 python bench.py --config C2 --no-cpu --no-e2e --steps 5 > gpurun_out/c2pin.json 2> gpurun_out/c2pin.err
python -c "import json; d=json.load(open('gpurun_out/c2pin.json')); print('C2', d['ms_per_step'], d['roofline_fp64']['frac'], 'fma', d['fma_mode']['ms_per_step'], 'validation', d['validation']['ms_per_step'])"
