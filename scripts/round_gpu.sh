#!/bin/bash
# Full GPU pass for a milestone: parity tests, smoke, bench (with CPU baseline
# and e2e), reference arm, launch list + one full ncu capture.  Logs -> gpurun_out/.
TAG=${TAG:-r1}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${TAG}_smoke.log
timeout 1500 python bench.py ${BENCH_ARGS} > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
if [ -z "$NO_REF" ]; then timeout 1200 python bench.py --impl reference --steps 3 --warmup 1 ${BENCH_ARGS} > gpurun_out/${TAG}_bench_ref.json 2> gpurun_out/${TAG}_bench_ref.err; fi
if [ -z "$NO_PROF" ]; then bash scripts/profile.sh ${TAG}_prof ${PROF_ARGS}; fi
tail -n 2 gpurun_out/${TAG}_pytest_gpu.log gpurun_out/${TAG}_smoke.log
