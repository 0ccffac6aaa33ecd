"""Per-mode MTTKRP time of the default HB-CSF plan (CUDA events, median of
10), with the plan's leaf-blocking / CSL-blocking info, for A/B sweeps of the
HBK_* knobs:  python scripts/mode_times.py nell-1 flickr-3d"""
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

import paper_1904_03329_b200 as hb
from paper_1904_03329_b200.generate import CONFIGS, config_tensor
from paper_1904_03329_b200.kernels import mttkrp_device, plan_for

tag = " ".join(f"{k}={v}" for k, v in sorted(__import__("os").environ.items()) if k.startswith("HBK_"))
for cfg in sys.argv[1:]:
    dims = CONFIGS[cfg]["dims"]
    t = config_tensor(cfg)
    f = [torch.rand((d, 32), device="cuda") for d in dims]
    tot = 0.0
    for mode in range(3):
        h = hb.split_fibers(hb.build_hbcsf(t, hb.allmode_order(dims, mode)), hb.SplitConfig())
        pl = plan_for(h, mode, 32)
        y, _ = mttkrp_device(h, f, mode)
        for _ in range(3):
            mttkrp_device(h, f, mode, out=y)
        ts = []
        for _ in range(10):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            mttkrp_device(h, f, mode, out=y)
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        ms = statistics.median(ts)
        tot += ms
        print(f"[{tag}] {cfg} mode {mode}: {ms:.3f} ms  leaf_blocks {pl.info.leaf_blocks} "
              f"blocked_nnz {pl.info.leaf_blocked_nnz} head_share {pl.info.leaf_head_share_ppm / 1e6:.3f} "
              f"csl_blocks {pl.info.csl_blocks} gather_rows {pl.info.gather_rows / 1e6:.1f}M", flush=True)
        del h, pl, y
        torch.cuda.empty_cache()
    print(f"[{tag}] {cfg} step {tot:.3f} ms", flush=True)
    del t, f
    torch.cuda.empty_cache()
