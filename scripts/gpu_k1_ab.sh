# K1 A/B over library variants: C2 and C1 bench lines. usage: bash scripts/gpu_k1_ab.sh "tag ..."
set -x
mkdir -p gpurun_out
run() {
  tag=$1; shift
  for i in 1 2; do
    env "$@" timeout 600 python bench.py --config C2 --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/k1v_${tag}_C2_$i.json 2>gpurun_out/k1v_${tag}.err; echo $tag rc=$?
  done
  env "$@" timeout 600 python bench.py --config C1 --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/k1v_${tag}_C1_1.json 2>>gpurun_out/k1v_${tag}.err; echo $tag C1 rc=$?
}
run default OSC_X=1
for v in $1; do run $v OSC_LIB=paper_1702_02207_b200/_variants/$v/libosc_b200.so; done
python - <<'PY'
import json,glob
for f in sorted(glob.glob('gpurun_out/k1v_*.json')):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1]); print(f, round(d['ms_per_step'],3), d['value'], d['clocks']['sm_mhz'], d['clocks']['reasons'])
    except Exception as e: print(f, 'ERR', e)
PY
