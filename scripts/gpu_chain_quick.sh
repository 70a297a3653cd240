# Quick check of a chain-kernel build: the chain parity/edge tests, then the C3 and C4 device times.
timeout 900 python -m pytest tests/test_gpu_edge.py tests/test_gpu_parity.py tests/test_gpu_validation.py tests/test_gpu_sharded.py -x -q -m gpu 2>&1 | tail -2
for c in C3 C4; do
  timeout 300 python bench.py --config $c --steps 3 --warmup 3 --no-cpu --no-e2e 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['config']['workload'][:2], round(d['ms_per_step'],2), round(d['roofline']['frac'],4))"
done
