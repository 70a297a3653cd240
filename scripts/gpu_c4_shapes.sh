# C4 whole-chain shapes (OSC_WHOLE) with the current builds.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu -k "chain or edge or hypothesis" > gpurun_out/pytest_chain.log 2>&1; echo pytest rc=$?; tail -1 gpurun_out/pytest_chain.log
for sh in default 4,256 8,128; do
  if [ $sh = default ]; then unset OSC_WHOLE; else export OSC_WHOLE=$sh; fi
  timeout 600 python bench.py --config C4 --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/c4s_${sh/,/x}.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/c4s_${sh/,/x}.json')); print('C4 $sh', round(d['ms_per_step'],2))"
done
