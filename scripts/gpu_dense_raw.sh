set -x
mkdir -p gpurun_out
timeout 600 python bench.py --config C5 --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/d_base.json 2>&1; echo rc=$?
OSC_DENSE_RAW=1 timeout 600 python bench.py --config C5 --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/d_raw.json 2>&1; echo rc=$?
for sh in "2,128" "2,256" "1,256" "4,128"; do OSC_B2=$sh timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/b2_${sh/,/x}.json 2>&1; echo $sh rc=$?; done
