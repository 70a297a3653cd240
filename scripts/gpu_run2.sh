# Round-1 measurement pass: tests, bench lines, tile-shape sweeps, ncu evidence.
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_gpu.log
for c in C2 C4 C3 C1; do timeout 600 python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo bench $c rc=$?; done
# tile-shape sweeps (no e2e / cpu legs)
for cfg in "8,256 32" "8,256 16" "8,128 16" "4,256 16" "4,256 32" "4,512 16" "4,512 32" "2,512 16" "8,256 64"; do
  set -- $cfg
  OSC_TILE=$1 timeout 300 python bench.py --config C3 --halo $2 --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/sweep_C3_${1/,/x}_T$2.json 2>&1; echo sweep C3 $cfg rc=$?
done
for w in "4,256" "8,128" "2,512"; do
  OSC_WHOLE=$w timeout 300 python bench.py --config C4 --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/sweep_C4_${w/,/x}.json 2>&1; echo sweep C4 $w rc=$?
done
# ncu: launch list of the C2 bench, then a full capture of the batch2 kernel
ARGS="--config C2 --steps 2 --warmup 3 --no-e2e --no-cpu"
python bench.py $ARGS > gpurun_out/ncu_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_C2.csv python bench.py $ARGS > gpurun_out/ncu_launch.log 2>&1; echo ncu1 rc=$?
ARGS1="--config C2 --steps 1 --warmup 3 --no-e2e --no-cpu"
python bench.py $ARGS1 > gpurun_out/ncu_plain1.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:batch2 -s 1 -c 1 -o gpurun_out/prof_batch2 python bench.py $ARGS1 > gpurun_out/ncu_full.log 2>&1; echo ncu2 rc=$?
ls -la gpurun_out
