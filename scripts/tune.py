"""Sweep kernel variants / task sizes on one generated tensor (GPU box).

    python scripts/tune.py --config nell-2 --var 0 1 2 --task 64 128 256
Prints per-mode mean kernel ms (CUDA events) and the sum."""
import argparse
import os
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import numpy as np
import torch

import paper_1904_03329_b200 as hb
from paper_1904_03329_b200.generate import CONFIGS, config_tensor
from paper_1904_03329_b200.kernels import _Plan, _device_factors

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="nell-2")
ap.add_argument("--scale", type=float, default=1.0)
ap.add_argument("--var", type=int, nargs="+", default=[0, 1, 2])
ap.add_argument("--task", type=int, nargs="+", default=[128])
ap.add_argument("--reps", type=int, default=10)
ap.add_argument("--check", action="store_true")
ap.add_argument("--heavy", nargs="+", default=["512:64:512"], help="H:tau:W of the heavy-slice layout (H=0 off)")
args = ap.parse_args()

cfg = CONFIGS[args.config]
dims = cfg["dims"]
t = config_tensor(args.config, scale=args.scale)
reps = [hb.split_fibers(hb.build_hbcsf(t, hb.allmode_order(dims, m)), hb.SplitConfig()) for m in range(3)]
rng = np.random.default_rng(cfg["seed"])
f = [torch.from_numpy(rng.random((d, 32))).float().cuda() for d in dims]
ref = None
import itertools
for var, task, hv in itertools.product(args.var, args.task, args.heavy):
        H, tau, W = hv.split(":")
        os.environ["HBK_HEAVY_H"], os.environ["HBK_HEAVY_TAU"], os.environ["HBK_HEAVY_W"] = H, tau, W
        os.environ["HBK_CSF_VARIANT"] = str(var)
        os.environ["HBK_TASK_NNZ"] = str(task)
        ms = []
        outs = []
        for m in range(3):
            h = reps[m]
            pl = _Plan(h.coo_part._dev().ptr if h.coo_part.nnz else None, h.csl_part._h.ptr,
                       h.csf_part._h.ptr, None, m, 32, dims[m])
            ptrs = _device_factors(f, m)[0]
            out = torch.empty((dims[m], 32), device="cuda")
            for _ in range(3):
                pl.execute(ptrs, out)
            ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.reps)]
            for a, b in ev:
                a.record()
                pl.execute(ptrs, out)
                b.record()
            torch.cuda.synchronize()
            ms.append(statistics.mean(a.elapsed_time(b) for a, b in ev))
            outs.append(out.clone())
        dev = ""
        if ref is None:
            ref = outs
        else:
            dev = max(float(((o - r).norm(dim=1) / (1 + r.norm(dim=1))).max()) for o, r in zip(outs, ref))
            dev = f" maxdev_vs_first={dev:.2e}"
        print(f"var={var} task={task} heavy={hv}: per-mode ms {[round(x, 4) for x in ms]} sum {sum(ms):.4f}{dev}", flush=True)
