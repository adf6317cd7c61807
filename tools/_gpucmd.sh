set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests_r2a.log 2>&1; tail -3 gpurun_out/gpu_tests_r2a.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-other-configs --no-slab-shares > gpurun_out/bench_r2a.json 2> gpurun_out/bench_r2a.err
python -c "import json; d=json.loads(open('gpurun_out/bench_r2a.json').read().strip().splitlines()[-1]); print(d['value'], d['stages_ms'], d['roofline']['frac'], d['latency_ms']['device_p50'])"
python tools/profile_bench_step.py 2 > gpurun_out/plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_pnn_tiles -s 1 -c 1 -o gpurun_out/tiles_f python tools/profile_bench_step.py 2 > gpurun_out/ncu_f.log 2>&1; tail -2 gpurun_out/ncu_f.log
