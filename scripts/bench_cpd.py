"""CP-ALS iteration benchmark (BASELINE.json configs[4]: nell-1-shaped, R=32,
MTTKRP of every mode + the NCCL factor-row all-gather).

    python scripts/bench_cpd.py [--config nell-1] [--iters 5] [--scale 1.0]
    torchrun --nproc-per-node N --master-addr 127.0.0.1 scripts/bench_cpd.py ...

One process per GPU; each rank owns an nnz-balanced row range of every mode
(paper_1904_03329_b200.distributed.cp_als_distributed).  Reports the median
ALS-sweep time (max over ranks: every sweep ends in collectives, so ranks
finish together) and the MTTKRP-equivalent GFLOP/s (3 modes x 3*nnz*R per
sweep).  Synthetic SURVEY Appendix-A tensor, generated on every rank.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

RANK = 32


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="nell-1")
    ap.add_argument("--iters", type=int, default=5)
    ap.add_argument("--scale", type=float, default=1.0)
    args = ap.parse_args()

    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0")) % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    backend = os.environ.get("HBK_BENCH_BACKEND", "nccl")
    if not dist.is_initialized():
        if world == 1:
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", "29533")
            os.environ.setdefault("RANK", "0")
            os.environ.setdefault("WORLD_SIZE", "1")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)

    from paper_1904_03329_b200.distributed import cp_als_distributed
    from paper_1904_03329_b200.generate import CONFIGS, config_tensor

    cfg = CONFIGS[args.config]
    t0 = time.perf_counter()
    t = config_tensor(args.config, scale=args.scale)
    torch.cuda.synchronize()
    gen_s = time.perf_counter() - t0
    # wall clock per sweep (host perf_counter around each sweep, through its
    # fit; exchanges, host bookkeeping and launch gaps included), median over
    # the sweeps after the first (which builds the plans); max over ranks.
    # The sum of mode_seconds (device spans) is reported beside it.
    walls = []
    tic = time.perf_counter()
    model, hist = cp_als_distributed(t, rank=RANK, max_iters=args.iters + 1, fit_tol=0.0,
                                     seed=cfg["seed"], sweep_hook=lambda it, s: walls.append(s))
    total_s = time.perf_counter() - tic
    sweeps = [sum(h.mode_seconds) for h in hist[2:]]
    tt = torch.tensor([statistics.median(walls[1:]), statistics.median(sweeps)],
                      dtype=torch.float64, device="cuda")
    dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    sweep, sweep_dev = float(tt[0]), float(tt[1])
    flops = 3 * 3.0 * t.nnz * RANK
    if rank == 0:
        print(json.dumps({
            "metric": "CP-ALS sweep (MTTKRP all modes + factor all-gather), MTTKRP-equivalent GFLOP/s",
            "value": flops / sweep / 1e9, "unit": "GFLOP/s", "ms_per_sweep": sweep * 1e3,
            "ms_per_sweep_mode_seconds": sweep_dev * 1e3,
            "timing": "host wall clock per sweep (median after the first), max over ranks",
            "sweep_wall_ms_all": [x * 1e3 for x in walls],
            "n_gpus": world, "iters": len(sweeps), "higher_is_better": True, "scaling": "strong",
            "dtype": "f32 MTTKRP, f64 ALS algebra",
            "config": {"workload": f"{args.config}-shaped CP-ALS R=32", "dims": list(cfg["dims"]),
                       "nnz": t.nnz, "scale": args.scale, "backend": backend},
            "fits": [h.fit for h in hist], "generate_s": gen_s, "total_s": total_s,
            "sweep_ms_all": [x * 1e3 for x in sweeps],
        }), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
