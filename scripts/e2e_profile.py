"""cProfile of the host-array MTTKRP path (bench e2e leg) on nell-2."""
import cProfile
import pstats
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

import paper_1904_03329_b200 as hb
from paper_1904_03329_b200.generate import CONFIGS, config_tensor

cfg = CONFIGS["nell-2"]
dims = cfg["dims"]
t = config_tensor("nell-2", scale=1.0)
reps = [hb.split_fibers(hb.build_hbcsf(t, hb.allmode_order(dims, m)), hb.SplitConfig()) for m in range(3)]
rng = np.random.default_rng(2)
f64 = [rng.random((d, 32)) for d in dims]
if "--pinned" in sys.argv:
    f64 = [torch.from_numpy(f).float().pin_memory() for f in f64]
for m in range(3):
    hb.mttkrp_hbcsf(reps[m], f64, m)
torch.cuda.synchronize()


def loop(k=10):
    for _ in range(k):
        for m in range(3):
            hb.mttkrp_hbcsf(reps[m], f64, m)


tic = time.perf_counter()
loop()
print("ms/step", (time.perf_counter() - tic) / 10 * 1e3)
pr = cProfile.Profile()
pr.enable()
loop()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
# device-side view: H2D, kernel, D2H per call
from torch.profiler import ProfilerActivity, profile
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    loop(3)
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=15))
