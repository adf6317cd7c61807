# Round evidence: full bench line, reference arm, launch list, ncu --set full of K1 / fan K1 / trilinear K1.
set -x
timeout 1200 python bench.py > gpurun_out/r2_bench.json 2> gpurun_out/r2_bench.err; tail -c 600 gpurun_out/r2_bench.json
timeout 900 python bench.py --impl reference > gpurun_out/r2_bench_reference.json 2> gpurun_out/r2_bench_reference.err; tail -c 300 gpurun_out/r2_bench_reference.json
python tools/profile_bench_step.py 2 > gpurun_out/plain.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches.csv python tools/profile_bench_step.py 2 > gpurun_out/ncu_l.log 2>&1
python tools/profile_bench_step.py 2 > gpurun_out/plain.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"k_pnn_tiles|k_tile_desc|k_pnn_work|k_fill_warp|k_depth|k_band" -s 6 -c 6 -o gpurun_out/r2_step python tools/profile_bench_step.py 2 > gpurun_out/ncu_s.log 2>&1
python tools/profile_config.py cfg3 2 > gpurun_out/p3.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"k_fan_tiles|k_fan_desc" -s 2 -c 2 -o gpurun_out/r2_fan python tools/profile_config.py cfg3 2 > gpurun_out/ncu_f.log 2>&1
python tools/profile_config.py cfg5 2 > gpurun_out/p5.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"k_insert" -s 1 -c 1 -o gpurun_out/r2_tri python tools/profile_config.py cfg5 2 > gpurun_out/ncu_t.log 2>&1
ls -la gpurun_out/r2_*
