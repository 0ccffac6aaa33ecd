"""Standalone MTTKRP at P GPUs, measured rank by rank on one B200.

The sharded MTTKRP has no collective in the timed region (bench.py --gpus N:
each rank owns a contiguous, nonzero-balanced row range of every mode and
runs its own HB-CSF plans; time = max over ranks).  So the N-GPU step time is
determined by the slowest rank's shard alone, and each rank's shard can be
built and timed on one GPU exactly as bench.py's rank r would build it
(bench.prepare with world = P, rank = r).  Prints, per config and P, every
rank's step time, the max (= the predicted P-GPU step), the whole-job
GFLOP/s and the strong-scaling efficiency against P = 1.

    python scripts/shard_scaling.py flickr-3d delicious-3d [--ps 2,4,8]
"""
import argparse
import json
import statistics
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import torch

import bench
from paper_1904_03329_b200 import shard
from paper_1904_03329_b200.generate import config_tensor


class RankEnv:
    """The subset of bench.Env that bench.prepare reads."""

    def __init__(self, world, rank):
        self.torch, self.world, self.rank = torch, world, rank


def step_ms(st, reps=20, warm=3):
    per_mode = []
    for m, plan in enumerate(st["plans"]):
        if plan is None:
            per_mode.append(0.0)
            continue
        for _ in range(warm):
            plan.execute(st["ptrs"][m], st["outs"][m])
        ts = []
        for _ in range(reps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            plan.execute(st["ptrs"][m], st["outs"][m])
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        per_mode.append(statistics.median(ts))
    return per_mode


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="+")
    ap.add_argument("--ps", default="2,4,8")
    a = ap.parse_args()
    args = argparse.Namespace(scale=1.0)
    out = {}
    for cfg in a.configs:
        t = config_tensor(cfg)
        nnz = t.nnz
        flops = 3 * 3.0 * nnz * bench.RANK
        st = bench.prepare(RankEnv(1, 0), cfg, args, tensor=t)
        one = step_ms(st)
        bench.free(st)
        res = {"nnz": nnz, "p1_ms": sum(one), "p1_per_mode_ms": one, "p1_gflops": flops / sum(one) / 1e6}
        print(f"{cfg} P=1: {sum(one):.3f} ms {res['p1_gflops']:.0f} GFLOP/s", flush=True)
        for P in [int(x) for x in a.ps.split(",")]:
            # pass 1: the static cost partition; pass 2: bench.prepare's
            # calibration (per-rank times -> shard.refine_row_ranges), here
            # with the ranks timed one after another instead of all-gathered
            override = None
            for pass_ in ("static", "calibrated"):
                ranks, all_ranges, costs = [], None, None
                for r in range(P):
                    st = bench.prepare(RankEnv(P, r), cfg, args, tensor=t, ranges=override)
                    pm = step_ms(st)
                    all_ranges, costs = st["all_ranges"], st["costs"]
                    shard_nnz = [c["coo_nnz"] + c["csl_nnz"] + c["csf_nnz"] if c else 0 for c in st["census"]]
                    ranks.append({"rank": r, "ms": sum(pm), "per_mode_ms": pm, "shard_nnz": shard_nnz,
                                  "rows": st["rows_local"], "census": st["census"]})
                    bench.free(st)
                worst = max(x["ms"] for x in ranks)
                eff = res["p1_ms"] / (P * worst)
                key = f"p{P}" if pass_ == "calibrated" else f"p{P}_static"
                res[key] = {"max_rank_ms": worst, "mean_rank_ms": statistics.mean(x["ms"] for x in ranks),
                            "gflops": flops / worst / 1e6, "strong_scaling_efficiency": eff,
                            "ranges": all_ranges, "ranks": ranks}
                print(f"{cfg} P={P} {pass_}: max rank {worst:.3f} ms (mean {res[key]['mean_rank_ms']:.3f}), "
                      f"{flops / worst / 1e6:.0f} GFLOP/s, efficiency {eff:.2f}", flush=True)
                if pass_ == "calibrated":
                    # bench.prepare keeps, per mode, the cut whose slowest rank is faster
                    st0, st1 = res[f"p{P}_static"]["ranks"], ranks
                    best = sum(min(max(x["per_mode_ms"][m] for x in st0), max(x["per_mode_ms"][m] for x in st1))
                               for m in range(3))
                    res[key]["kept_max_ms_bound"] = best
                    print(f"{cfg} P={P} kept (per-mode better cut): slowest-rank sum {best:.3f} ms, "
                          f"efficiency {res['p1_ms'] / (P * best):.2f}", flush=True)
                override = [shard.refine_row_ranges(costs[m], all_ranges[m], [x["per_mode_ms"][m] for x in ranks])
                            for m in range(3)]
        out[cfg] = res
        del t
        torch.cuda.empty_cache()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
