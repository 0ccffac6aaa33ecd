"""Touched-rows exchange volume of row-sharded CP-ALS (SURVEY §8e asks for
the measured union sizes): for P ranks with nnz-balanced row ranges per mode,
rank r needs the rows of factor d that its shards of the *other* modes read;
it owns range_d[r] itself.  Prints, per P, the factor-row ingress per GPU per
sweep for the touched-rows exchange vs full replication (max and mean over
ranks), emulating the ranks one after another on one GPU.

    python scripts/exchange_volume.py nell-1 2 4 8
"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

from paper_1904_03329_b200 import shard
from paper_1904_03329_b200.generate import CONFIGS, config_tensor

R = 32


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "nell-1"
    Ps = [int(x) for x in sys.argv[2:]] or [2, 4, 8]
    dims = CONFIGS[cfg]["dims"]
    t = config_tensor(cfg)
    idx = torch.from_numpy(np.ascontiguousarray(t.indices).astype(np.int64)).cuda()
    hists = [shard.slice_histogram(t, m).cpu().numpy() for m in range(3)]
    out = {"config": cfg, "rank": R, "per_P": {}}
    for P in Ps:
        ranges = [shard.plan_row_ranges(hists[m], P) for m in range(3)]
        touched, full = [], []
        for r in range(P):
            rows_in = 0
            for d in range(3):
                need = []
                for n in range(3):
                    if n == d:
                        continue
                    lo, hi = ranges[n][r]
                    sel = (idx[:, n] >= lo) & (idx[:, n] < hi)
                    need.append(idx[sel, d])
                u = torch.unique(torch.cat(need))
                lo, hi = ranges[d][r]
                rows_in += int(((u < lo) | (u >= hi)).sum())
            touched.append(rows_in * R * 4)
            full.append(sum((dims[d] - (ranges[d][r][1] - ranges[d][r][0])) for d in range(3)) * R * 4)
        rec = {"touched_GB_max": max(touched) / 1e9, "touched_GB_mean": float(np.mean(touched)) / 1e9,
               "full_GB_max": max(full) / 1e9, "full_GB_mean": float(np.mean(full)) / 1e9}
        out["per_P"][P] = rec
        print(f"{cfg} P={P}: ingress per GPU per sweep: touched {rec['touched_GB_mean']:.2f} GB mean / "
              f"{rec['touched_GB_max']:.2f} max; full replication {rec['full_GB_mean']:.2f} / "
              f"{rec['full_GB_max']:.2f} GB", flush=True)
    Path("gpurun_out").mkdir(exist_ok=True)
    Path(f"gpurun_out/exchange_volume_{cfg}.json").write_text(json.dumps(out, indent=1) + "\n")


if __name__ == "__main__":
    main()
