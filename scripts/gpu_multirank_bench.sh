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
# A rank failing inside the sharded C3 side record must cost the sub-record only:
# the C2 line is still printed (once), every rank exits 0.
for fr in 1 0; do
  P=$((P+1))
  OSC_BENCH_FAIL_RANK=$fr OSC_SHARDED_C3_LIMIT=60 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $P \
    bench.py --gpus 2 --config C2 --steps 1 --warmup 3 --no-e2e > gpurun_out/mr_fail$fr.json 2> gpurun_out/mr_fail$fr.err; echo fail-rank $fr rc=$?
  python -c "import json;L=open('gpurun_out/mr_fail$fr.json').read().strip().splitlines();d=json.loads(L[-1]);print('fail-rank $fr: lines', len(L), d['n_gpus'], d['value'], d['sharded_c3'])"
done
# A rank that stalls: every rank's watchdog ends it, rank 0 prints the line it has.
P=$((P+1))
OSC_BENCH_STALL_RANK=1 OSC_SHARDED_C3_LIMIT=45 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $P \
  bench.py --gpus 2 --config C2 --steps 1 --warmup 3 --no-e2e > gpurun_out/mr_stall1.json 2> gpurun_out/mr_stall1.err; echo stall-rank 1 rc=$?
python -c "import json;L=open('gpurun_out/mr_stall1.json').read().strip().splitlines();d=json.loads(L[-1]);print('stall-rank 1: lines', len(L), d['n_gpus'], d['value'], d['sharded_c3'])"
