#!/bin/bash
# per-launch kernel times and counters (ncu, serialized) of the bench's plan
# executions, per config; summarise with scripts/kind_summary.py
mkdir -p gpurun_out
for c in ${CONFIGS:-nell-2 flickr-3d delicious-3d nell-1}; do
  ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_active,lts__t_sector_hit_rate.pct,dram__bytes_read.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:k_mttkrp3 --csv \
    python bench.py --config $c --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --also "" --cpd none --no-amortize > gpurun_out/kind_$c.csv 2>&1
done
