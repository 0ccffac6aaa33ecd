#!/bin/bash
# ncu counters of the CSF kernel variants on nell-2 mode 0 (one launch each).
mkdir -p gpurun_out
M="gpu__time_duration.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,l1tex__throughput.avg.pct_of_peak_sustained_active,lts__throughput.avg.pct_of_peak_sustained_elapsed,l1tex__t_sector_hit_rate.pct,lts__t_sector_hit_rate.pct,dram__bytes_read.sum,smsp__average_warp_latency_issue_stalled_long_scoreboard,smsp__pcsamp_warps_issue_stalled_long_scoreboard,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,l1tex__data_bank_reads.avg.pct_of_peak_sustained_elapsed,l1tex__m_xbar2l1tex_read_bytes.sum,smsp__inst_executed_op_ldgsts.sum"
for v in ${VARIANTS:-0 2}; do
  HBK_CSF_VARIANT=$v ncu --metrics $M --clock-control none -k regex:k_mttkrp3 -c 1 --csv \
    python scripts/tune.py --config nell-2 --var $v --task 128 --reps 1 > gpurun_out/ncu_var$v.csv 2>&1
done
