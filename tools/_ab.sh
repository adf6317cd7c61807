# A/B of compile variants: bench insert stage for each lib in abtmp/ (and the default), interleaved
for rep in 1 2 3; do
for L in default abtmp/*.so; do
  if [ "$L" = default ]; then unset SVR_LIB_PATH; else export SVR_LIB_PATH=$PWD/$L; fi
    timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-other-configs --no-slab-shares > gpurun_out/ab.json 2>/dev/null
    python -c "import json,sys; d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]); print(sys.argv[1], round(d['value'],1), round(d['stages_ms']['insert'],4), round(d['roofline']['frac'],3))" $L
done
done
