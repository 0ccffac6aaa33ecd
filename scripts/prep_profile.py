"""Where does preprocessing time go?  Per mode: build_hbcsf, split_fibers, the
census accessors, plan creation (synchronised wall clock per stage).

    python scripts/prep_profile.py nell-1
"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

import paper_1904_03329_b200 as hb
from paper_1904_03329_b200.generate import CONFIGS, config_tensor
from paper_1904_03329_b200.kernels import plan_for


def tick():
    torch.cuda.synchronize()
    return time.perf_counter()


cfg = sys.argv[1] if len(sys.argv) > 1 else "nell-1"
dims = CONFIGS[cfg]["dims"]
t = config_tensor(cfg)
torch.cuda.synchronize()
for rep in range(2):
    for mode in range(3):
        mo = hb.allmode_order(dims, mode)
        t0 = tick()
        h = hb.build_hbcsf(t, mo)
        t1 = tick()
        hs = hb.split_fibers(h, hb.SplitConfig())
        t2 = tick()
        census = (hs.coo_part.nnz, hs.csl_part.num_slices, hs.csl_part.nnz, hs.csf_part.num_slices,
                  hs.csf_part.num_fibers, hs.csf_part.nnz)
        t3 = tick()
        plan = plan_for(hs, mode, 32)
        t4 = tick()
        print(f"rep {rep} mode {mode}: build_hbcsf {t1 - t0:.3f}s split {t2 - t1:.3f}s "
              f"census {t3 - t2:.3f}s plan {t4 - t3:.3f}s  (heavy tasks {plan.info.tasks_heavy}, "
              f"zero rows {plan.info.tasks_zero})", flush=True)
