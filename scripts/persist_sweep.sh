#!/bin/bash
mkdir -p gpurun_out
for c in ${CONFIGS:-nell-1 flickr-3d}; do
  for pm in ${PERSIST:-0 40 80 200}; do
    for hmb in ${HOTS:-80}; do
      echo "persist=$pm hot_mb=$hmb" >> gpurun_out/persist_$c.txt
      HBK_PERSIST_MB=$pm HBK_HOT_MB=$hmb timeout 600 python scripts/tune.py --config $c --var 2 --task 128 --heavy 128:32:2048 >> gpurun_out/persist_$c.txt 2>&1
    done
  done
done
