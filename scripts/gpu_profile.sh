# ncu evidence for every hot kernel (run under gpurun; one GPU).  Each ncu run
# follows the same command exiting 0 without ncu (B200_PROFILING.md).
#   bash scripts/gpu_profile.sh            -> gpurun_out/prof_*.ncu-rep + launches_C2.csv
set -x
mkdir -p gpurun_out
ARGS="--config C2 --steps 2 --warmup 3 --no-e2e --no-cpu --no-side"
python bench.py $ARGS > gpurun_out/plain_c2.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_C2.csv python bench.py $ARGS > gpurun_out/ncu_launch.log 2>&1; echo launches rc=$?
ARGS1="--config C2 --steps 1 --warmup 3 --no-e2e --no-cpu --no-side"
python bench.py $ARGS1 > gpurun_out/plain_c2b.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:batch2 -s 1 -c 1 -o gpurun_out/prof_batch2 python bench.py $ARGS1 > gpurun_out/ncu_b2.log 2>&1; echo batch2 rc=$?
python scripts/prof_chain.py C3 96 > gpurun_out/plain_c3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:chain_tiles_persistent -s 1 -c 1 -o gpurun_out/prof_c3 python scripts/prof_chain.py C3 96 > gpurun_out/ncu_c3.log 2>&1; echo c3 rc=$?
python scripts/prof_chain.py C4 1024 > gpurun_out/plain_c4.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:chain_rk4 -s 1 -c 1 -o gpurun_out/prof_c4 python scripts/prof_chain.py C4 1024 > gpurun_out/ncu_c4.log 2>&1; echo c4 rc=$?
python scripts/prof_dense.py 3 > gpurun_out/plain_c5.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:dense_rk4_gemm -s 2 -c 1 -o gpurun_out/prof_dense python scripts/prof_dense.py 3 > gpurun_out/ncu_c5.log 2>&1; echo c5 rc=$?
