# ptxas option variants (scripts/build_variants.py) on C2 / C4 / C3.
mkdir -p gpurun_out
for v in default rul2 rul8 rul10 O2; do
  if [ $v = default ]; then unset OSC_LIB; else export OSC_LIB=$PWD/paper_1702_02207_b200/_variants/$v/libosc_b200.so; fi
  for c in C2 C4 C3; do
    timeout 300 python bench.py --config $c --no-cpu --no-e2e --steps 3 > gpurun_out/pv_${v}_$c.json 2> gpurun_out/pv_${v}_$c.err
    python -c "import json; d=json.load(open('gpurun_out/pv_${v}_$c.json')); print('$v $c', round(d['ms_per_step'],2), round(d['roofline_fp64']['frac'],3))"
  done
done
