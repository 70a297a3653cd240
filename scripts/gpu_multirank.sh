# Multi-rank path check on a one-GPU box: 2 ranks over gloo sharing cuda:0.
set -x
mkdir -p gpurun_out
export OSC_BENCH_BACKEND=gloo
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 --steps 3 --warmup 3 > gpurun_out/mr_C2.json 2> gpurun_out/mr_C2.err; echo C2 rc=$?
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29518 bench.py --gpus 2 --config C3 --steps 2 --warmup 3 > gpurun_out/mr_C3.json 2> gpurun_out/mr_C3.err; echo C3 rc=$?
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29519 bench.py --impl reference --gpus 2 --steps 1 --warmup 3 > gpurun_out/mr_ref.json 2> gpurun_out/mr_ref.err; echo ref rc=$?
tail -3 gpurun_out/mr_C2.err gpurun_out/mr_C3.err
