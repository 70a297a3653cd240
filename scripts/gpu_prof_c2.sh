set -x
mkdir -p gpurun_out
ARGS1="--config C2 --steps 1 --warmup 3 --no-e2e --no-cpu"
python bench.py $ARGS1 > gpurun_out/ncu_plain1.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:batch2 -s 1 -c 1 -o gpurun_out/prof_batch2_v2 python bench.py $ARGS1 > gpurun_out/ncu_full.log 2>&1; echo ncu rc=$?
