"""Host-array MTTKRP call time (pinned fp32 factors in, float64 rows out) on
nell-2, against the device time of the same call's kernel."""
import statistics
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

import paper_1904_03329_b200 as hb
from paper_1904_03329_b200 import kernels as K
from paper_1904_03329_b200.generate import CONFIGS, config_tensor

dims = CONFIGS["nell-2"]["dims"]
t = config_tensor("nell-2")
reps = [hb.build_hbcsf(t, hb.allmode_order(dims, m)) for m in range(3)]
rng = np.random.default_rng(2)
fp = [torch.from_numpy(rng.random((d, 32))).float().pin_memory() for d in dims]
for m in range(3):
    hb.mttkrp_hbcsf(reps[m], fp, m)
torch.cuda.synchronize()
t0 = time.perf_counter()
for it in range(10):
    for m in range(3):
        hb.mttkrp_hbcsf(reps[m], fp, m)
print(f"api call  {(time.perf_counter() - t0) / 30 * 1e3:7.3f} ms")
dev = [torch.from_numpy(np.asarray(f)).cuda() for f in fp]
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
ev[0].record()
for it in range(10):
    for m in range(3):
        hb.mttkrp_device(reps[m], dev, m)
ev[1].record()
torch.cuda.synchronize()
print(f"device    {ev[0].elapsed_time(ev[1]) / 30:7.3f} ms")
