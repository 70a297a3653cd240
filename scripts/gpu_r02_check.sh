# Round-2 check: sharded/multirank tests, bench N=1 line, multi-rank bench path over gloo.
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_sharded.py tests/test_gpu_multirank.py -q -x > gpurun_out/pytest_sh.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_sh.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo bench rc=$?
OSC_BENCH_BACKEND=gloo timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29541 bench.py --gpus 2 --steps 2 --warmup 3 --no-e2e > gpurun_out/bench_gloo2.json 2> gpurun_out/bench_gloo2.err; echo bench2 rc=$?
tail -c 3000 gpurun_out/bench_gloo2.json
