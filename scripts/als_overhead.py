"""Where does a CP-ALS sweep's time go beyond the kernels?  torch.profiler
over sweeps of cp_als (R=32 fused path) on a config: device kernel time vs
wall time per sweep, and the top host-side entries."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from torch.profiler import ProfilerActivity, profile

import paper_1904_03329_b200 as hb
from paper_1904_03329_b200.generate import config_tensor

cfg = sys.argv[1] if len(sys.argv) > 1 else "nell-2"
t = config_tensor(cfg)
hb.cp_als(t, rank=32, max_iters=2, fit_tol=0.0, seed=1)  # plans built
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    t0 = time.perf_counter()
    m, h = hb.cp_als(t, rank=32, max_iters=5, fit_tol=0.0, seed=1)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
print(cfg, "sweep ms", [round(sum(x.mode_seconds) * 1e3, 3) for x in h[1:]], "wall total ms", round(wall * 1e3, 2))
ka = prof.key_averages()
dev = sum(e.self_device_time_total for e in ka) / 1e3
print("device self time total ms", round(dev, 3))
print(ka.table(sort_by="self_cpu_time_total", row_limit=18))
print(ka.table(sort_by="self_device_time_total", row_limit=10))
