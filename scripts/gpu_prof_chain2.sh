set -x
mkdir -p gpurun_out
python scripts/prof_chain.py C3 96 > gpurun_out/prof_c3_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:chain_tiles_persistent -s 1 -c 1 -o gpurun_out/prof_c3p python scripts/prof_chain.py C3 96 > gpurun_out/ncu_c3.log 2>&1; echo ncu3 rc=$?
python scripts/prof_chain.py C4 1024 > gpurun_out/prof_c4_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:chain_rk4 -s 1 -c 1 -o gpurun_out/prof_c4b python scripts/prof_chain.py C4 1024 > gpurun_out/ncu_c4.log 2>&1; echo ncu4 rc=$?
ARGS="--config C2 --steps 2 --warmup 3 --no-e2e --no-cpu"
python bench.py $ARGS > gpurun_out/ncu_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_C2.csv python bench.py $ARGS > gpurun_out/ncu_launch.log 2>&1; echo ncu1 rc=$?
