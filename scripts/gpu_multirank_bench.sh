# The bench's multi-rank paths over gloo on one GPU (path checks, not scaling numbers).
set -x
mkdir -p gpurun_out
export OSC_BENCH_BACKEND=gloo
P=29610
for cfg in "C2 3" "C4 2" "C5 2" "C3 2"; do
  set -- $cfg
  P=$((P+1))
  timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node $2 --master-addr 127.0.0.1 --master-port $P \
    bench.py --gpus $2 --config $1 --steps 1 --warmup 3 --no-e2e > gpurun_out/mr_$1_$2.json 2> gpurun_out/mr_$1_$2.err; echo $1 $2 rc=$?
  python -c "import json;d=json.loads(open('gpurun_out/mr_$1_$2.json').read().strip().splitlines()[-1]);print('$1', d['n_gpus'], d['value'], d['ms_per_step'], d['config'].get('parallelism'), d.get('sharded_c3',{}) and {k:d['sharded_c3'].get(k) for k in ('ms_per_step','host_us_per_period_max','error')})"
done
