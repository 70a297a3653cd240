# K5 check: dense tests (restatement, analytic, ragged shapes, full C5 64 steps), C5 bench line, ncu.
set -x
mkdir -p gpurun_out
TAG=${TAG:-tma}
timeout 1200 python -m pytest tests/test_gpu_dense.py tests/test_gpu_fullsize.py -k "dense or c5" -q -x > gpurun_out/pytest_dense_$TAG.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_dense_$TAG.log
timeout 600 python -m pytest tests/test_gpu_hypothesis.py -k dense -q -x > gpurun_out/pytest_dense_hyp_$TAG.log 2>&1; echo hyp rc=$?
tail -2 gpurun_out/pytest_dense_hyp_$TAG.log
timeout 900 python bench.py --config C5 --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/C5_$TAG.json 2> gpurun_out/C5_$TAG.err; echo bench rc=$?
python -c "import json;d=json.loads(open('gpurun_out/C5_$TAG.json').read().strip().splitlines()[-1]);print(d['ms_per_step'], d['roofline']['achieved'], d['roofline']['frac'], d['roofline'].get('cublas_dgemm_tflops'), d['clocks'])"
python scripts/prof_dense.py 3 > gpurun_out/plain_c5.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:dense_rk4_gemm -s 2 -c 1 -o gpurun_out/prof_dense_$TAG python scripts/prof_dense.py 3 > gpurun_out/ncu_c5.log 2>&1; echo ncu rc=$?
