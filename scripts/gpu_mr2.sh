set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_multirank.py -x -q > gpurun_out/pytest_mr.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_mr.log
export OSC_BENCH_BACKEND=gloo
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29519 bench.py --impl reference --gpus 2 --steps 1 --warmup 3 > gpurun_out/mr_ref.json 2> gpurun_out/mr_ref.err; echo ref rc=$?
cat gpurun_out/mr_ref.json
