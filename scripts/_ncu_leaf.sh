mkdir -p gpurun_out
M="dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sectors.sum,lts__t_sectors_lookup_hit.sum"
HBK_LEAF_BLOCK_MB=0 ncu --metrics $M -k regex:k_mttkrp3 -c 40 --csv --log-file gpurun_out/leaf_ncu_off.csv python scripts/mode_times.py nell-1 > /dev/null 2>&1
ncu --metrics $M -k regex:k_mttkrp3 -c 60 --csv --log-file gpurun_out/leaf_ncu_on.csv python scripts/mode_times.py nell-1 > /dev/null 2>&1
ncu --metrics $M -k regex:k_mttkrp3 -c 60 --csv --log-file gpurun_out/leaf_ncu_del.csv python scripts/mode_times.py delicious-3d > /dev/null 2>&1
