# K1 with longer chunks between divergence checks (scripts/build_variants.py c128 c256): C2 and C1.
run() {
  timeout 300 python bench.py --config C2 --no-cpu --no-e2e --no-side --steps 6 > gpurun_out/k1_$1.json 2> gpurun_out/k1_$1.err
  python -c "import json; d=json.load(open('gpurun_out/k1_$1.json')); print('$1 C2', round(min(d['step_ms']),3), round(d['ms_per_step'],3))"
  timeout 300 python bench.py --config C1 --no-cpu --no-e2e --steps 3 > gpurun_out/k1c1_$1.json 2> gpurun_out/k1c1_$1.err
  python -c "import json; d=json.load(open('gpurun_out/k1c1_$1.json')); print('$1 C1', round(d['ms_per_step'],3))"
}
mkdir -p gpurun_out
run default
for v in ${VARIANTS:-c128 c256}; do OSC_LIB=$PWD/paper_1702_02207_b200/_variants/$v/libosc_b200.so run $v; done
