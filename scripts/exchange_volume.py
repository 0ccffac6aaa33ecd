"""Touched-rows exchange volume of row-sharded CP-ALS (SURVEY §8e asks for
the measured union sizes): for P ranks with the row ranges cp_als_distributed
uses (shard.partition_costs: nonzeros + fibers + a per-row charge),
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
# single-GPU per-mode MTTKRP and row-update seconds (bench / scripts/bench_cpd.py,
# profiles/r1s10_*): the compute of one sweep, divided by P in the model
MODEL = {"nell-1": ([2.63e-3, 2.64e-3, 3.03e-3], [0.22e-3, 0.16e-3, 1.73e-3])}


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "nell-1"
    Ps = [int(x) for x in sys.argv[2:]] or [2, 4, 8]
    dims = CONFIGS[cfg]["dims"]
    t = config_tensor(cfg)
    idx = torch.from_numpy(np.ascontiguousarray(t.indices).astype(np.int64)).cuda()
    hists = [shard.partition_costs(t, m).cpu().numpy() for m in range(3)]
    out = {"config": cfg, "rank": R, "per_P": {}}
    for P in Ps:
        ranges = [shard.plan_row_ranges(hists[m], P) for m in range(3)]
        touched, full = [], []
        crit = np.zeros((P, 3))  # bytes of factor d the next mode (d+1) reads, received by rank r
        rest = np.zeros((P, 3))  # bytes only later modes read (SplitExchange's deferred part)
        for r in range(P):
            rows_in = 0
            for d in range(3):
                by = {}
                for n in range(3):
                    if n == d:
                        continue
                    lo, hi = ranges[n][r]
                    sel = (idx[:, n] >= lo) & (idx[:, n] < hi)
                    by[n] = torch.unique(idx[sel, d])
                u = torch.unique(torch.cat(list(by.values())))
                lo, hi = ranges[d][r]
                remote = lambda x: x[(x < lo) | (x >= hi)]  # noqa: E731
                rows_in += int(remote(u).numel())
                c = remote(by[(d + 1) % 3])
                later = remote(by[(d + 2) % 3])
                crit[r, d] = c.numel() * R * 4
                rest[r, d] = int((~torch.isin(later, c)).sum()) * R * 4
            touched.append(rows_in * R * 4)
            full.append(sum((dims[d] - (ranges[d][r][1] - ranges[d][r][0])) for d in range(3)) * R * 4)
        rec = {"touched_GB_max": max(touched) / 1e9, "touched_GB_mean": float(np.mean(touched)) / 1e9,
               "full_GB_max": max(full) / 1e9, "full_GB_mean": float(np.mean(full)) / 1e9,
               "critical_GB_max_per_factor": (crit.max(0) / 1e9).tolist(),
               "deferred_GB_max_per_factor": (rest.max(0) / 1e9).tolist()}
        # sweep model (max over ranks, ingress-bound exchange at BW): mode m =
        # MTTKRP_m/P + update_m/P, then factor m's critical rows; factor m's
        # deferred rows overlap mode m+1's compute, any excess stalls
        if MODEL.get(cfg):
            mt, up = MODEL[cfg]
            for bw in (700e9, 900e9):
                worst_plain = worst_split = 0.0
                for r in range(P):
                    plain = split = 0.0
                    for m in range(3):
                        comp = (mt[m] + up[m]) / P
                        plain += comp + (crit[r, m] + rest[r, m]) / bw
                        prev_rest = rest[r, (m - 1) % 3] / bw
                        split += comp + crit[r, m] / bw + max(0.0, prev_rest - comp)
                    worst_plain, worst_split = max(worst_plain, plain), max(worst_split, split)
                rec[f"model_sweep_ms_{int(bw / 1e9)}GBs"] = {"touched": worst_plain * 1e3,
                                                              "touched_split": worst_split * 1e3}
        out["per_P"][P] = rec
        print(f"{cfg} P={P}: ingress per GPU per sweep: touched {rec['touched_GB_mean']:.2f} GB mean / "
              f"{rec['touched_GB_max']:.2f} max; full replication {rec['full_GB_mean']:.2f} / "
              f"{rec['full_GB_max']:.2f} GB; model {json.dumps({k: v for k, v in rec.items() if k.startswith('model')})}",
              flush=True)
    Path("gpurun_out").mkdir(exist_ok=True)
    Path(f"gpurun_out/exchange_volume_{cfg}.json").write_text(json.dumps(out, indent=1) + "\n")


if __name__ == "__main__":
    main()
