#!/bin/bash
# The paper's format comparison (HB-CSF vs B-CSF vs CSF vs COO) on the GPU:
#   bash scripts/format_compare.sh nell-2 flickr-3d ...   (on the GPU box)
mkdir -p gpurun_out
for c in "$@"; do
  for f in hbcsf bcsf csf coo; do
    python bench.py --config $c --format $f --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --also "" --cpd none --no-amortize 2>/dev/null | tail -1 > gpurun_out/fmt_${c}_${f}.json
    python - "$c" "$f" <<'PY'
import json, sys
c, f = sys.argv[1], sys.argv[2]
d = json.load(open(f"gpurun_out/fmt_{c}_{f}.json"))
g = d["roofline"].get("gather") or {}
print(f"{c:13s} {f:6s} {d['ms_per_step']:8.3f} ms/step {d['value']:9.1f} GFLOP/s  per-mode {[round(x, 3) for x in d['roofline']['per_mode_ms']]}  gather-frac {g.get('frac')}  clocks {d['clocks']['sm_mhz']} {d['clocks']['reasons']}")
PY
  done
done
