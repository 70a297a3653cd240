# K5 (C5 dense) under ptxas option variants of the whole library (scripts/build_variants.py rul2 rul8 rul10 O2).
run() {
  timeout 600 python bench.py --config C5 --no-cpu --no-e2e --steps 2 > gpurun_out/k5_$1.json 2> gpurun_out/k5_$1.err
  python -c "import json; d=json.load(open('gpurun_out/k5_$1.json')); print('$1', round(d['ms_per_step'],1), round(d['roofline']['frac'],4))"
}
mkdir -p gpurun_out
run default
for v in rul2 rul8 rul10 O2; do OSC_LIB=$PWD/paper_1702_02207_b200/_variants/$v/libosc_b200.so run $v; done
