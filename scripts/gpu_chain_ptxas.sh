# Chain kernels (C3, C4) under ptxas option variants of the whole library (scripts/build_variants.py).
run() {
  for c in C3 C4; do
    timeout 300 python bench.py --config $c --no-cpu --no-e2e --steps 3 > gpurun_out/ch_$1_$c.json 2> gpurun_out/ch_$1_$c.err
    python -c "import json; d=json.load(open('gpurun_out/ch_$1_$c.json')); print('$1', '$c', round(d['ms_per_step'],2))"
  done
}
mkdir -p gpurun_out
run default
for v in ${VARIANTS:-rul3 rul4 rul6 rul7}; do OSC_LIB=$PWD/paper_1702_02207_b200/_variants/$v/libosc_b200.so run $v; done
