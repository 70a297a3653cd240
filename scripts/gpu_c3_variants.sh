# C3 A/B over library variants (scripts/build_variants.py) + ncu of the default K3 launch.
# usage: bash scripts/gpu_c3_variants.sh "tag1 tag2 ..." [ncu]
set -x
mkdir -p gpurun_out
run() {  # tag, env...
  tag=$1; shift
  for i in 1 2; do
    env "$@" timeout 600 python bench.py --config C3 --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/c3v_${tag}_$i.json 2>gpurun_out/c3v_${tag}.err; echo $tag rc=$?
  done
}
run default OSC_X=1
run div3 OSC_DIV2=0
for v in $1; do run $v OSC_LIB=paper_1702_02207_b200/_variants/$v/libosc_b200.so; done
python - <<'PY'
import json,glob
for f in sorted(glob.glob('gpurun_out/c3v_*_*.json')):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1]); print(f, round(d['ms_per_step'],2), d['clocks']['sm_mhz'], d['clocks']['reasons'])
    except Exception as e: print(f, 'ERR', e)
PY
if [ "$2" = ncu ]; then
python scripts/prof_chain.py C3 96 > gpurun_out/plain_c3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:chain_tiles_persistent -s 1 -c 1 -o gpurun_out/prof_c3_d2 python scripts/prof_chain.py C3 96 > gpurun_out/ncu_c3.log 2>&1; echo ncu rc=$?
fi
