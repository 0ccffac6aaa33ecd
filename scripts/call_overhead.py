"""Fixed per-call cost of the host-array MTTKRP (tiny tensor, pinned fp32
factors in, float64 rows out): Python + ctypes + copies + one sync."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import cProfile
import pstats

import numpy as np
import torch

import paper_1904_03329_b200 as hb

rng = np.random.default_rng(0)
dims = (50, 40, 30)
idx = np.stack([rng.integers(0, d, 300) for d in dims], 1).astype(np.uint32)
t = hb.canonicalize(hb.CooTensor(dims, idx, rng.random(300)))
h = hb.build_hbcsf(t, (0, 1, 2))
f = [torch.from_numpy(rng.random((d, 32))).float().pin_memory() for d in dims]
for _ in range(50):
    hb.mttkrp_hbcsf(h, f, 0)
torch.cuda.synchronize()
n = 2000
t0 = time.perf_counter()
for _ in range(n):
    hb.mttkrp_hbcsf(h, f, 0)
print(f"per call {1e6 * (time.perf_counter() - t0) / n:.1f} us")
pr = cProfile.Profile()
pr.enable()
for _ in range(500):
    hb.mttkrp_hbcsf(h, f, 0)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(14)
