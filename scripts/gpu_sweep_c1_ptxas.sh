# C1 latency across ptxas option variants (scripts/build_variants.py).
mkdir -p gpurun_out
for v in default rul2 rul8 rul10 O2; do
  if [ $v = default ]; then unset OSC_LIB; else export OSC_LIB=$PWD/paper_1702_02207_b200/_variants/$v/libosc_b200.so; fi
  timeout 300 python bench.py --config C1 --no-cpu --no-e2e --steps 3 > gpurun_out/c1v_$v.json 2> gpurun_out/c1v_$v.err
  python -c "import json; d=json.load(open('gpurun_out/c1v_$v.json')); print('$v', round(d['ms_per_step'],2), 'validation', round(d['validation']['ms_per_step'],2))"
done
