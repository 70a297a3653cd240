run() {
  timeout 300 python bench.py --config C2 --no-cpu --no-e2e --no-side --steps 10 > gpurun_out/k1_$1.json 2> gpurun_out/k1_$1.err
  python -c "import json; d=json.load(open('gpurun_out/k1_$1.json')); print('$1', round(d['ms_per_step'],3), 'validation', round(d['validation']['ms_per_step'],2))"
}
for rep in 1 2; do
run default
for v in u1 u2 u3; do OSC_LIB=$PWD/paper_1702_02207_b200/_variants/$v/libosc_b200.so run $v; done
done
