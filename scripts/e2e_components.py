"""Where the host-array call's time goes (nell-2, the reference calling
convention: NumPy float64 factors in, NumPy float64 rows out).

Per mode: the whole call; the f64->f32 conversion into page-locked staging
alone (pool, several chunk sizes / worker counts); the host-to-device copy
of the staged factors; the kernel; the device->host copy of the rows."""
import statistics
import sys
import time
from concurrent.futures import ThreadPoolExecutor
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
f64 = [rng.random((d, 32)) for d in dims]


def wall(fn, n=20):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(n):
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    return statistics.median(ts) * 1e3


print("host:", open("/proc/cpuinfo").read().count("processor\t"), "cpus", flush=True)
for m in range(3):
    print(f"mode {m}: call {wall(lambda: hb.mttkrp_hbcsf(reps[m], f64, m)):.3f} ms", flush=True)

# conversion alone
src = [f64[d] for d in (1, 2)]
stage = [torch.empty(a.shape, dtype=torch.float32, pin_memory=True) for a in src]
sv = [s.numpy() for s in stage]
for workers in (1, 4, 8, 16):
    pool = ThreadPoolExecutor(workers)
    for chunk in (256 << 10, 1 << 20, 4 << 20):
        jobs = []
        for i, a in enumerate(src):
            step = max(1, chunk // (a.shape[1] * 8))
            jobs += [(i, r, min(a.shape[0], r + step)) for r in range(0, a.shape[0], step)]

        def run():
            fs = [pool.submit(np.copyto, sv[i][r0:r1], src[i][r0:r1], casting="unsafe") for i, r0, r1 in jobs]
            for f in fs:
                f.result()

        print(f"convert mode-0 factors (9.7 MB f64): workers {workers:2d} chunk {chunk >> 10:5d} KB "
              f"{wall(run):.3f} ms", flush=True)
    pool.shutdown()

# single-thread memcpy and conversion bandwidth
a = f64[2]
b = np.empty_like(a)
print(f"1-thread f64 memcpy 7.4 MB: {wall(lambda: np.copyto(b, a)):.3f} ms", flush=True)
print(f"1-thread f64->f32 7.4 MB: {wall(lambda: np.copyto(sv[1], a, casting='unsafe')):.3f} ms", flush=True)

# H2D of the staged fp32 factors, D2H of the rows
dev = [torch.empty(s.shape, dtype=torch.float32, device="cuda") for s in stage]


def h2d():
    for d_, s in zip(dev, stage):
        d_.copy_(s, non_blocking=True)


print(f"H2D pinned fp32 4.9 MB: {wall(h2d):.3f} ms", flush=True)
src64 = [torch.from_numpy(x) for x in src]


def h2d_pageable64():
    for d_, s in zip(dev, src64):
        d_.copy_(s.to("cuda", non_blocking=False).float())


print(f"H2D pageable fp64 9.7 MB + device cast: {wall(h2d_pageable64):.3f} ms", flush=True)
y = torch.empty((dims[2], 32), dtype=torch.float64, device="cuda")
hy = torch.empty((dims[2], 32), dtype=torch.float64, pin_memory=True)
print(f"D2H pinned fp64 7.4 MB: {wall(lambda: hy.copy_(y, non_blocking=True)):.3f} ms", flush=True)
print(f"pinned alloc 7.4 MB: {wall(lambda: torch.empty((dims[2], 32), dtype=torch.float64, pin_memory=True)):.3f} ms", flush=True)
devf = [torch.from_numpy(x).float().cuda() for x in f64]
for m in range(3):
    print(f"mode {m}: device call {wall(lambda: K.mttkrp_device(reps[m], devf, m)):.3f} ms", flush=True)

# instrumented calls: wall time per phase of the real call
import collections

acc = collections.defaultdict(list)


def timed_method(obj, name, label, sync=False):
    fn = getattr(obj, name)

    def w(*a, **k):
        if sync:
            torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = fn(*a, **k)
        if sync:
            torch.cuda.synchronize()
        acc[label].append(time.perf_counter() - t0)
        return r

    setattr(obj, name, w)


st = K._host_stage()
timed_method(st, "upload_all", "upload_all (sync after)", sync=True)
timed_method(st, "download", "download")
timed_method(K._Plan, "execute", "execute (sync after)", sync=True)
timed_method(K, "_nonfinite_flags", "nonfinite")
timed_method(K, "_check_factors", "check")
for it in range(20):
    for m in range(3):
        t0 = time.perf_counter()
        hb.mttkrp_hbcsf(reps[m], f64, m)
        acc[f"call mode {m} (instrumented)"].append(time.perf_counter() - t0)
for k, v in acc.items():
    print(f"{k:36s} median {statistics.median(v[2:]) * 1e3:.3f} ms  n={len(v)}", flush=True)
