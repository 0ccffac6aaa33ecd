"""MTTKRP time per mode vs rank R on a config tensor (fast path at R=32,
generic kernel otherwise)."""
import statistics
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
reps = [hb.build_hbcsf(t, hb.allmode_order(dims, m)) for m in range(3)]
for R in [int(x) for x in (sys.argv[2:] or ["8", "16", "32", "64", "128"])]:
    f = [torch.rand((d, R), device="cuda") for d in dims]
    ms = []
    for m in range(3):
        mttkrp_device(reps[m], f, m)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(5):
            mttkrp_device(reps[m], f, m)
        b.record()
        torch.cuda.synchronize()
        ms.append(a.elapsed_time(b) / 5)
    flops = 3 * 3.0 * t.nnz * R
    print(f"{cfg} R={R}: per-mode ms {[round(x, 3) for x in ms]}  {flops / (sum(ms) * 1e-3) / 1e9:.0f} GFLOP/s", flush=True)
