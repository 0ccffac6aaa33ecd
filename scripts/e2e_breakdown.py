"""Per-call timeline of the host-array MTTKRP (pinned fp32 factors in,
float64 rows out) on nell-2: host time per phase, averaged over calls."""
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
ph = {k: [] for k in ("check", "plan", "upload", "launch", "d2h+sync", "widen", "flags", "total")}
for it in range(20):
    for m in range(3):
        t0 = time.perf_counter()
        r = K._check_factors(reps[m].dims, fp, m, check_finite="staged")
        t1 = time.perf_counter()
        plan = K.plan_for(reps[m], m, r)
        t2 = time.perf_counter()
        ptrs, keep, on_dev, checks = K._device_factors(fp, m)
        t3 = time.perf_counter()
        y = plan.execute(ptrs)
        t4 = time.perf_counter()
        st = K._host_stage()
        buf = st._pinned(torch, ("out",), y.numel(), y.dtype)
        buf[: y.numel()].view(y.shape).copy_(y, non_blocking=True)
        torch.cuda.current_stream().synchronize()
        t5 = time.perf_counter()
        out = np.empty(tuple(y.shape))
        np.copyto(out, buf.numpy()[: y.numel()].reshape(y.shape))
        t6 = time.perf_counter()
        for d, ok in checks:
            bool(ok)
        t7 = time.perf_counter()
        for k, a, b in (("check", t0, t1), ("plan", t1, t2), ("upload", t2, t3), ("launch", t3, t4),
                        ("d2h+sync", t4, t5), ("widen", t5, t6), ("flags", t6, t7), ("total", t0, t7)):
            ph[k].append((b - a) * 1e3)
for k, v in ph.items():
    print(f"{k:10s} {statistics.median(v):7.3f} ms")
