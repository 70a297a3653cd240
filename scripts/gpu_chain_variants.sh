# C3 + C4 over library variants (scripts/build_variants.py). usage: bash scripts/gpu_chain_variants.sh "tag ..."
set -x
mkdir -p gpurun_out
run() {
  tag=$1; shift
  for c in C3 C4; do
    env "$@" timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/chv_${tag}_$c.json 2>gpurun_out/chv_${tag}.err; echo $tag $c rc=$?
  done
}
run default OSC_X=1
run div3 OSC_DIV2=0
for v in $1; do run $v OSC_LIB=paper_1702_02207_b200/_variants/$v/libosc_b200.so; done
python - <<'PY'
import json,glob
for f in sorted(glob.glob('gpurun_out/chv_*.json')):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1]); print(f, round(d['ms_per_step'],2), d['clocks']['sm_mhz'], d['clocks']['reasons'])
    except Exception as e: print(f, 'ERR', e)
PY
