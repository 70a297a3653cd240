# ncu evidence for K1 (batch2) after a change: launch list of a C2 bench run
# and one --set full capture of the hot kernel.  Each ncu run follows the same
# command exiting 0 without ncu (B200_PROFILING.md).
set -x
mkdir -p gpurun_out
ARGS="--config C2 --steps 2 --warmup 3 --no-e2e --no-cpu --no-side"
python bench.py $ARGS > gpurun_out/plain_c2.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_C2.csv python bench.py $ARGS > gpurun_out/ncu_launch.log 2>&1; echo launches rc=$?
ARGS1="--config C2 --steps 1 --warmup 3 --no-e2e --no-cpu --no-side"
ncu --set full --clock-control none --import-source on -k regex:batch2_rk4 -s 1 -c 1 -o gpurun_out/prof_batch2 python bench.py $ARGS1 > gpurun_out/ncu_b2.log 2>&1; echo batch2 rc=$?
