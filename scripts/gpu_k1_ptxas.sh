# K1 (C2) under ptxas option variants of the whole library (scripts/build_variants.py rul2 rul8 rul10 O2).
run() {
  timeout 300 python bench.py --config C2 --no-cpu --no-e2e --no-side --steps 6 > gpurun_out/k1_$1.json 2> gpurun_out/k1_$1.err
  python -c "import json; d=json.load(open('gpurun_out/k1_$1.json')); print('$1', round(min(d['step_ms']),3), round(d['ms_per_step'],3), 'validation', round(d['validation']['ms_per_step'],2))"
}
mkdir -p gpurun_out
run default
for v in ${VARIANTS:-rul2 rul8 rul10 O2}; do OSC_LIB=$PWD/paper_1702_02207_b200/_variants/$v/libosc_b200.so run $v; done
