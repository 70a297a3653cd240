# Host-pointer path change: its GPU tests, then C2/C4 e2e lines.
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_c_abi.py -x -q -m gpu -k "host or c_program" > gpurun_out/pt_host.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pt_host.log
for c in C2 C4 C3; do
  timeout 400 python bench.py --config $c --no-cpu --steps 3 > gpurun_out/bh_$c.json 2> gpurun_out/bh_$c.err; echo $c rc=$?
  python -c "import json; d=json.load(open('gpurun_out/bh_$c.json')); print('$c', '%.4g'%d['value'], 'e2e %.4g'%d['e2e']['value'], round(d['e2e']['value']/d['value'],3))"
done
