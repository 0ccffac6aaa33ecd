#!/bin/bash
# L1 / L2 / crossbar counters of the MTTKRP launches of one config (bench.py
# under ncu, the 3 launches after warm-up).  Usage: bash scripts/ncu_l1l2.sh <tag> <config> [bench args]
TAG=$1; CFG=$2; shift 2
M="gpu__time_duration.sum,sm__cycles_elapsed.avg,lts__cycles_elapsed.avg"
M="$M,l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum"
M="$M,l1tex__t_sectors_pipe_lsu_mem_global_op_ld_lookup_hit.sum,l1tex__m_xbar2l1tex_read_bytes.sum"
M="$M,l1tex__m_xbar2l1tex_read_bytes_mem_lg_op_ld.sum,lts__t_sectors_srcunit_tex_op_read.sum"
M="$M,lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum,lts__t_sectors.sum,lts__t_bytes.sum"
M="$M,l1tex__data_pipe_lsu_wavefronts.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"
M="$M,l1tex__data_bank_reads.sum,l1tex__lsu_writeback_active.sum,lts__throughput.avg.pct_of_peak_sustained_elapsed"
M="$M,l1tex__throughput.avg.pct_of_peak_sustained_active,l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed"
M="$M,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active"
mkdir -p gpurun_out
ncu --metrics $M --clock-control none -k regex:k_mttkrp3 -s 3 -c 3 --csv --log-file gpurun_out/${TAG}_l1l2.csv \
    python bench.py --config $CFG --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --also "" --cpd none --no-amortize "$@" > gpurun_out/${TAG}_l1l2.log 2>&1
echo "ncu rc=$?"
