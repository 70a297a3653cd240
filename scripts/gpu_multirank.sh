# Multi-rank path check on a one-GPU box: 2 ranks over gloo sharing cuda:0.
set -x
mkdir -p gpurun_out
export OSC_BENCH_BACKEND=gloo
run() { timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $1 bench.py --gpus 2 "${@:2}"; }
run 29517 --steps 3 --warmup 3 > gpurun_out/mr_C2.json 2> gpurun_out/mr_C2.err; echo C2 rc=$?
run 29518 --config C3 --steps 2 --warmup 3 > gpurun_out/mr_C3.json 2> gpurun_out/mr_C3.err; echo C3 rc=$?
run 29520 --config C3 --transport peer --steps 2 --warmup 3 > gpurun_out/mr_C3p.json 2> gpurun_out/mr_C3p.err; echo C3 peer rc=$?
run 29519 --impl reference --steps 1 --warmup 3 > gpurun_out/mr_ref.json 2> gpurun_out/mr_ref.err; echo ref rc=$?
