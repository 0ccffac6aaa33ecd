"""torch.profiler view of CP-ALS sweeps (nell-1, R=32) to see where the
non-MTTKRP time goes."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from torch.profiler import ProfilerActivity, profile

import paper_1904_03329_b200 as hb
from paper_1904_03329_b200.generate import config_tensor

t = config_tensor(sys.argv[1] if len(sys.argv) > 1 else "nell-1")
hb.cp_als(t, rank=32, max_iters=1, fit_tol=0.0, seed=1)  # plans built, warm
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    hb.cp_als(t, rank=32, max_iters=3, fit_tol=0.0, seed=1)
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=25))
print(prof.key_averages().table(sort_by="cpu_time_total", row_limit=25))
