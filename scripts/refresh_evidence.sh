#!/bin/bash
# Round-end evidence on one B200 (run under gpurun): DRAM traffic per mode for
# every config, one ncu full capture of the nell-2 kernel + its launch list,
# bench lines for all configs, the reference arm and the CP-ALS sweeps.
#   bash scripts/refresh_evidence.sh <tag>
TAG=${1:-r1s7}
set -x
mkdir -p gpurun_out
python scripts/ncu_traffic.py nell-2 flickr-3d delicious-3d nell-1 > gpurun_out/traffic.log 2>&1
cp gpurun_out/ncu_summary.json profiles/ncu_summary.json 2>/dev/null
bash scripts/profile.sh ${TAG}_nell2 --config nell-2
python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
for c in flickr-3d delicious-3d nell-1; do
  python bench.py --config $c --no-cpu-baseline > gpurun_out/${TAG}_bench_$c.json 2>gpurun_out/${TAG}_bench_$c.err
done
python bench.py --impl reference > gpurun_out/${TAG}_bench_ref.json 2>&1
for c in nell-1 nell-2; do python scripts/bench_cpd.py --config $c > gpurun_out/${TAG}_cpd_$c.json 2>/dev/null; done
tail -c 300 gpurun_out/traffic.log
