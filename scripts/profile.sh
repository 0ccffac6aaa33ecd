#!/bin/bash
# ncu launch list + one full capture of the MTTKRP kernel (1 GPU).  Usage:
#   bash scripts/profile.sh <tag> <bench args...>
TAG=${1:-prof}; shift
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --also "" --cpd none --no-amortize "$@" > gpurun_out/${TAG}_launches.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_mttkrp3 -s 3 -c 3 \
    -o gpurun_out/${TAG} python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --also "" --cpd none --no-amortize "$@" > gpurun_out/${TAG}_full.log 2>&1
echo "profile rc=$?"
