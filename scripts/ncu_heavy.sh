#!/bin/bash
# ncu counters of the CSF kernel, heavy layout off/on (nell-2 mode 0)
mkdir -p gpurun_out
M="gpu__time_duration.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,l1tex__throughput.avg.pct_of_peak_sustained_active,lts__throughput.avg.pct_of_peak_sustained_elapsed,l1tex__t_sector_hit_rate.pct,lts__t_sector_hit_rate.pct,dram__bytes_read.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,l1tex__data_bank_reads.avg.pct_of_peak_sustained_elapsed,l1tex__m_xbar2l1tex_read_bytes.sum,smsp__inst_executed_op_ldgsts.sum,l1tex__lsu_writeback_active.avg.pct_of_peak_sustained_active,l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_active,l1tex__f_wavefronts.avg.pct_of_peak_sustained_active,lts__t_sectors.avg.pct_of_peak_sustained_elapsed,lts__d_sectors.avg.pct_of_peak_sustained_elapsed,l1tex__m_l1tex2xbar_req.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active,smsp__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active"
for hv in ${HEAVY:-0:64:512 512:64:2048}; do
  ncu --metrics $M --clock-control none -k regex:k_mttkrp3 -c 2 --csv \
    python scripts/tune.py --config nell-2 --var 0 --task 128 --reps 1 --heavy $hv > gpurun_out/ncu_heavy_${hv//:/_}.csv 2>&1
done
