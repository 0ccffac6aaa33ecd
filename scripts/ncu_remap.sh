#!/bin/bash
# DRAM / L2 / L1 counters of the remap-blocking probe's MTTKRP launches.
# Usage: bash scripts/ncu_remap.sh <tag> <config> <mode> <B|C> <nb list>
TAG=$1; shift
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct"
M="$M,l1tex__t_sector_hit_rate.pct,lts__t_bytes.sum,l1tex__m_xbar2l1tex_read_bytes.sum"
M="$M,l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"
mkdir -p gpurun_out
ncu --metrics $M --clock-control none -k regex:k_mttkrp3 --csv --log-file gpurun_out/${TAG}.csv \
    python scripts/remap_block_probe.py "$@" 1 > gpurun_out/${TAG}.log 2>&1
echo "ncu rc=$?"
