set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "chain or c3 or c4" > gpurun_out/pytest_chain.log 2>&1; echo pytest rc=$?
OSC_CHAIN_MINB=3 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "chain or c3 or c4" > gpurun_out/pytest_chain3.log 2>&1; echo pytest3 rc=$?
tail -2 gpurun_out/pytest_chain.log gpurun_out/pytest_chain3.log
for mb in 1 3; do
for c in C3 C4; do
OSC_CHAIN_MINB=$mb timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_${c}_minb$mb.json 2>&1; echo $c $mb rc=$?
done; done
