#!/bin/bash
# ncu counters of the sweep kernel variants on C4 (diagnostics): usage tools/shadow_prof.sh TAG
TAG=${1:-x}
M=gpu__time_duration.sum,sm__cycles_elapsed.max,l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,l1tex__t_sector_hit_rate.pct,l1tex__data_pipe_lsu_wavefronts.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum,l1tex__throughput.avg.pct_of_peak_sustained_elapsed,l1tex__m_l1tex2xbar_req_cycles_active.avg.pct_of_peak_sustained_elapsed,l1tex__m_xbar2l1tex_read_sectors.sum,lts__throughput.avg.pct_of_peak_sustained_elapsed,lts__t_sectors.sum,lts__t_sector_hit_rate.pct,lts__t_sectors_srcunit_tex_op_read.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,smsp__issue_active.avg.per_cycle_active,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio,smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio,smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio,smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio,smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio,smsp__average_warps_issue_stalled_wait_per_issue_active.ratio,l1tex__lsu_writeback_active.avg.pct_of_peak_sustained_elapsed,l1tex__f_wavefronts.sum,l1tex__t_set_conflicts_pipe_lsu_mem_global_op_ld.sum,launch__shared_mem_config_size
for v in 0 1; do
  timeout 900 ncu --metrics $M --clock-control none -k regex:k_sweep -c 1 --csv \
    --log-file gpurun_out/ncu_${TAG}_s$v.csv python tools/shadow_prof.py 4 $v 40 \
    > gpurun_out/ncu_${TAG}_s$v.log 2>&1
done
