"""MTTKRP time with a BlockSchedule (mttkrp_scheduled / mttkrp_hbcsf(schedule=),
the reference CLI's --threads path) vs the default plan, per mode."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

import paper_1904_03329_b200 as hb
from paper_1904_03329_b200.generate import CONFIGS, config_tensor
from paper_1904_03329_b200.kernels import mttkrp_device

cfg = sys.argv[1] if len(sys.argv) > 1 else "nell-2"
dims = CONFIGS[cfg]["dims"]
t = config_tensor(cfg)
f = [torch.rand((d, 32), device="cuda") for d in dims]
sc = hb.SplitConfig()


def timed(fn, n=10):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n


for mode in range(3):
    h = hb.split_fibers(hb.build_hbcsf(t, hb.allmode_order(dims, mode)), sc)
    s = hb.assign_slice_blocks(h.csf_part, sc)
    t0 = timed(lambda: mttkrp_device(h, f, mode))
    t1 = timed(lambda: mttkrp_device(h, f, mode, schedule=s))
    print(f"{cfg} mode {mode}: default {t0:.3f} ms, scheduled ({len(s.multiplicities)} slices, "
          f"{s.num_blocks} units) {t1:.3f} ms", flush=True)
