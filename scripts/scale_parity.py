"""At-scale oracle parity evidence: every mode of configs 2-5 on whole-slice
shards of >= 10M nonzeros (tests/scale_parity_lib.py).  Writes a JSON summary.

    python scripts/scale_parity.py [--target 10000000] [--out gpurun_out/r2_scale_parity.json]
"""
import argparse
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

from scale_parity_lib import run_config  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--target", type=int, default=10_000_000)
ap.add_argument("--configs", default="nell-2,flickr-3d,delicious-3d,nell-1")
ap.add_argument("--out", default=str(ROOT / "gpurun_out" / "r2_scale_parity.json"))
args = ap.parse_args()
recs = []
for c in args.configs.split(","):
    recs += run_config(c, args.target, seed=23, log=lambda s: print(s, flush=True))
    Path(args.out).parent.mkdir(parents=True, exist_ok=True)
    Path(args.out).write_text(json.dumps({"target_nnz": args.target, "tolerance": 1e-4,
                                          "records": recs}, indent=1))
ok = all(r["bit_exact"] and r["opcount_exact"] and r["max_row_dev"] <= 1e-4
         and r["max_row_dev_scheduled"] <= 1e-4 for r in recs)
print("scale parity:", "PASS" if ok else "FAIL")
sys.exit(0 if ok else 1)
