set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sharded.py -x -q -k "chain or c3 or c4 or local or tiled" > gpurun_out/pytest_chain.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_chain.log
timeout 600 python bench.py --config C3 --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_C3_persist.json 2>&1; echo c3 rc=$?
OSC_NO_PERSIST=1 timeout 600 python bench.py --config C3 --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_C3_nopersist.json 2>&1; echo c3np rc=$?
for T in 24 32; do timeout 600 python bench.py --config C3 --halo $T --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_C3_persist_T$T.json 2>&1; echo c3 T$T rc=$?; done
