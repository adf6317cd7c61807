# cfg5 trilinear K1 on 620 frames wholly inside a 19 GB slab: live timing, then ncu counters
# (selected metrics: few replay passes over the 19 GB volume) and source-level stall samples.
set -x
python tools/profile_config.py cfg5mid 3 > gpurun_out/p5m.log 2>&1 || { tail -5 gpurun_out/p5m.log; exit 1; }
tail -1 gpurun_out/p5m.log
M=gpu__time_duration.sum,smsp__inst_executed.sum,sm__issue_active.avg.pct_of_peak_sustained_elapsed,sm__warps_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,lts__t_sector_hit_rate.pct,launch__registers_per_thread,lts__t_requests_srcunit_tex_op_red.sum,lts__t_sectors_srcunit_tex_op_red.sum,lts__t_sectors_srcunit_tex_op_red_lookup_hit.sum,l1tex__t_requests_pipe_lsu_mem_global_op_red.sum,smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio,smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio,smsp__average_warps_issue_stalled_wait_per_issue_active.ratio,smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio,smsp__average_warps_issue_stalled_drain_per_issue_active.ratio,smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,lts__t_sectors_op_read.sum,lts__t_sectors_op_write.sum,lts__throughput.avg.pct_of_peak_sustained_elapsed
timeout 900 ncu --metrics $M --clock-control none -k regex:"k_insert" -s 1 -c 1 --csv --log-file gpurun_out/r2_tri_mid.csv python tools/profile_config.py cfg5mid 2 > gpurun_out/ncu_tm.log 2>&1
tail -3 gpurun_out/ncu_tm.log
timeout 900 ncu --section SourceCounters --section WarpStateStats --import-source on --clock-control none -k regex:"k_insert" -s 1 -c 1 -o gpurun_out/r2_tri_mid_src python tools/profile_config.py cfg5mid 2 > gpurun_out/ncu_tm2.log 2>&1
ls -la gpurun_out/r2_tri_mid*
