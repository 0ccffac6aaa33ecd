#!/bin/bash
# L2 hot-row budget sweep (HBK_HOT_MB) per config, CSF variant 2
mkdir -p gpurun_out
for c in ${CONFIGS:-nell-2 flickr-3d delicious-3d nell-1}; do
  for hmb in ${HOTS:-100000 80 40}; do
    echo "hot_mb=$hmb" >> gpurun_out/hot_$c.txt
    HBK_HOT_MB=$hmb timeout 600 python scripts/tune.py --config $c --var 2 --task 128 --heavy 128:32:2048 >> gpurun_out/hot_$c.txt 2>&1
  done
done
