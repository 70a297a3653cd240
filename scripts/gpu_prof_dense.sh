set -x
mkdir -p gpurun_out
python scripts/prof_dense.py 3 > gpurun_out/prof_dense_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:dense_rk4_gemm -s 2 -c 1 -o gpurun_out/prof_dense python scripts/prof_dense.py 3 > gpurun_out/ncu_dense.log 2>&1; echo ncu rc=$?
tail -3 gpurun_out/ncu_dense.log
