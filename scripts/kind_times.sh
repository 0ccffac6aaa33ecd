#!/bin/bash
# per-launch kernel times (ncu, serialized) of one plan execution per mode, per config
mkdir -p gpurun_out
for c in ${CONFIGS:-nell-2 flickr-3d delicious-3d nell-1}; do
  ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_active,lts__t_sector_hit_rate.pct,dram__bytes_read.sum,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:k_mttkrp3 --csv \
    python scripts/tune.py --config $c --var ${VAR:-2} --task 128 --reps 1 > gpurun_out/kind_$c.csv 2>&1
done
