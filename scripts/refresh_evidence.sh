set -x
python scripts/ncu_traffic.py nell-2 flickr-3d delicious-3d nell-1 > gpurun_out/traffic.log 2>&1
cp gpurun_out/ncu_summary.json profiles/ncu_summary.json 2>/dev/null
python bench.py > gpurun_out/r1s6_bench.json 2> gpurun_out/r1s6_bench.err
for c in flickr-3d delicious-3d nell-1; do python bench.py --config $c --no-cpu-baseline > gpurun_out/r1s6_bench_$c.json 2>gpurun_out/r1s6_bench_$c.err; done
python bench.py --impl reference > gpurun_out/r1s6_bench_ref.json 2>&1
tail -c 300 gpurun_out/traffic.log
