# Round evidence, part 1: GPU test suite + ncu --set full of the bench step's kernels, the fan K1
# and the trilinear K1 (each capture only after the same command exited 0 without ncu).
set -x
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r2_gpu_tests.log 2>&1; tail -3 gpurun_out/r2_gpu_tests.log
python tools/profile_bench_step.py 2 > gpurun_out/plain.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"k_pnn_tiles|k_tile_desc|k_pnn_work|k_fill_warp|k_depth|k_band" -s 6 -c 6 -o gpurun_out/r2_step python tools/profile_bench_step.py 2 > gpurun_out/ncu_s.log 2>&1
python tools/profile_config.py cfg3 2 > gpurun_out/p3.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"k_fan_tiles|k_fan_desc" -s 2 -c 2 -o gpurun_out/r2_fan python tools/profile_config.py cfg3 2 > gpurun_out/ncu_f.log 2>&1
python tools/profile_config.py cfg5 2 > gpurun_out/p5.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"k_insert|k_tri_warp" -s 1 -c 1 -o gpurun_out/r2_tri python tools/profile_config.py cfg5 2 > gpurun_out/ncu_t.log 2>&1
ls -la gpurun_out/r2_*
