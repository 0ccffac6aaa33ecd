"""Per-mode MTTKRP time with and without the zero fill of rows no bucket owns
(skip_unowned=True leaves them unwritten), to size the zero-row tasks' share:
    python scripts/zero_cost_probe.py flickr-3d nell-1"""
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

import paper_1904_03329_b200 as hb
from paper_1904_03329_b200.generate import CONFIGS, config_tensor
from paper_1904_03329_b200.kernels import mttkrp_device, plan_for


def timed(h, f, mode, **kw):
    y, _ = mttkrp_device(h, f, mode, **kw)
    for _ in range(3):
        mttkrp_device(h, f, mode, out=y, **kw)
    ts = []
    for _ in range(10):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        mttkrp_device(h, f, mode, out=y, **kw)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts)


for cfg in sys.argv[1:]:
    dims = CONFIGS[cfg]["dims"]
    t = config_tensor(cfg)
    f = [torch.rand((d, 32), device="cuda") for d in dims]
    for mode in range(3):
        h = hb.split_fibers(hb.build_hbcsf(t, hb.allmode_order(dims, mode)), hb.SplitConfig())
        pl = plan_for(h, mode, 32)
        owned = int(pl.owned_rows().numel())
        a = timed(h, f, mode)
        b = timed(h, f, mode, skip_unowned=True)
        print(f"{cfg} mode {mode}: rows {dims[mode]} owned {owned} (unowned "
              f"{(dims[mode] - owned) * 128 / 1e9:.2f} GB of zeros): {a:.3f} ms, "
              f"without the zero fill {b:.3f} ms", flush=True)
        del h, pl
        torch.cuda.empty_cache()
    del t, f
    torch.cuda.empty_cache()
