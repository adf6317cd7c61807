# Round evidence, part 2 (part 1: tools/_evidence_ncu.sh): full bench line, reference arm, ncu
# launch list of the bench step.
set -x
timeout 1200 python bench.py > gpurun_out/r2_bench.json 2> gpurun_out/r2_bench.err; tail -c 600 gpurun_out/r2_bench.json
timeout 900 python bench.py --impl reference > gpurun_out/r2_bench_reference.json 2> gpurun_out/r2_bench_reference.err; tail -c 300 gpurun_out/r2_bench_reference.json
python tools/profile_bench_step.py 2 > gpurun_out/plain.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches.csv python tools/profile_bench_step.py 2 > gpurun_out/ncu_l.log 2>&1
ls -la gpurun_out/r2_*
