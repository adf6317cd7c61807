# A/B of compile variants: bench stages for each lib in abtmp/ (and the default), interleaved
for rep in 1 2 3; do
for L in default abtmp/*.so; do
  if [ "$L" = default ]; then unset SVR_LIB_PATH; else export SVR_LIB_PATH=$PWD/$L; fi
    timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-other-configs --no-slab-shares > gpurun_out/ab.json 2>/dev/null
    python -c "import json,sys; d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]); s=d['stages_ms']; print(sys.argv[1], round(d['value'],1), 'ins', round(s['insert'],4), 'fill', round(s['fill'],4), 'rend', round(s['render'],4), round(d['roofline']['frac'],3), 'p50', round(d['latency_ms']['device_p50'],4))" $L
done
done
