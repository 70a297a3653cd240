# K1 (C2) sweep: step-loop unroll variants (scripts/build_variants.py u1 u2 u8)
# and launch shapes (OSC_B2), default library otherwise.
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_compare.py -x -q -m gpu > gpurun_out/pytest_k1.log 2>&1; echo pytest rc=$?; tail -1 gpurun_out/pytest_k1.log
run() {  # tag
  timeout 300 python bench.py --config C2 --no-cpu --no-e2e --no-side --steps 5 > gpurun_out/k1_$1.json 2> gpurun_out/k1_$1.err
  python -c "import json; d=json.load(open('gpurun_out/k1_$1.json')); print('$1', round(d['ms_per_step'],2), 'validation', round(d['validation']['ms_per_step'],2), 'fma', round(d['fma_mode']['ms_per_step'],2))"
}
run default
for v in u1 u2 u8; do OSC_LIB=$PWD/paper_1702_02207_b200/_variants/$v/libosc_b200.so run $v; done
for sh in 2,128 4,128 4,64 1,256; do OSC_B2=$sh run shape_${sh/,/x}; done
