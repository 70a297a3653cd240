for mode in nvml nvml smi; do
  if [ $mode = smi ]; then export OSC_BENCH_SMI=1; else unset OSC_BENCH_SMI; fi
  timeout 300 python bench.py --config C2 --no-cpu --no-e2e --no-side --steps 20 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read()); s=d['step_ms']; print('$mode', round(d['ms_per_step'],3), 'min', round(min(s),3), 'max', round(max(s),3), 'outliers', sum(1 for x in s if x>min(s)+0.5), d['clocks'])"
done
