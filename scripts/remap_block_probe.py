"""Would range-blocking a factor cut the DRAM traffic of the HBM-resident
configurations?  Emulates a blocked MTTKRP with the existing kernels: the
output-mode index is remapped to i' = block(x) * dims[mode] + i, where x is
the B (fiber) or C (leaf) index and block() cuts its rows into ``nb``
contiguous ranges.  The MTTKRP of the remapped tensor visits the nonzeros
block by block (slices are block-major), so every block's factor rows are
reused out of L2 — the access pattern of a blocked plan — and its output
(nb partial row sets) sums to the true rows.  Times per mode vs nb, and
checks the summed rows against the unblocked ones.

  python scripts/remap_block_probe.py delicious-3d 0 B 1,2,4,6,8
"""
import math
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import ctypes as C

import torch

import paper_1904_03329_b200 as hb
from paper_1904_03329_b200 import _native as N
from paper_1904_03329_b200.generate import CONFIGS, config_tensor
from paper_1904_03329_b200.kernels import mttkrp_device, plan_for

R = 32


def timed(h, f, mode, reps=10):
    y, _ = mttkrp_device(h, f, mode)
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        mttkrp_device(h, f, mode, out=y)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts), y


def main():
    cfg, mode, which = sys.argv[1], int(sys.argv[2]), sys.argv[3]
    nbs = [int(x) for x in sys.argv[4].split(",")]
    reps = int(sys.argv[5]) if len(sys.argv) > 5 else 10
    dims = CONFIGS[cfg]["dims"]
    t = config_tensor(cfg)
    idx = torch.empty((t.nnz, 3), dtype=torch.int32, device="cuda")
    vals = torch.empty(t.nnz, dtype=torch.float64, device="cuda")
    N.call("hbk_coo_export_device", t._dev().ptr, C.c_void_p(idx.data_ptr()),
           C.c_void_p(vals.data_ptr()), None, N.stream_ptr())
    mo = hb.allmode_order(dims, mode)
    x = mo[1] if which == "B" else mo[2]
    g = torch.Generator(device="cuda").manual_seed(1)
    f = [torch.rand((d, R), device="cuda", generator=g) for d in dims]
    base = None
    for nb in nbs:
        bs = math.ceil(dims[x] / nb)
        if nb == 1:
            h = hb.split_fibers(hb.build_hbcsf(t, mo), hb.SplitConfig())
            ms, y = timed(h, f, mode, reps)
            base = y.double()
            print(f"{cfg} mode {mode} nb=1: {ms:.3f} ms  (launches {plan_for(h, mode, R).info.launches})",
                  flush=True)
            del h
            continue
        new = idx.clone()
        new[:, mode] = (idx[:, x] // bs) * dims[mode] + idx[:, mode]
        d2 = list(dims)
        d2[mode] = nb * dims[mode]
        t2 = hb.canonicalize(hb.CooTensor(tuple(d2), new, vals))
        h2 = hb.split_fibers(hb.build_hbcsf(t2, mo), hb.SplitConfig())
        f2 = list(f)
        f2[mode] = torch.empty((d2[mode], R), device="cuda")
        ms, y2 = timed(h2, f2, mode, reps)
        ys = y2.view(nb, dims[mode], R).double().sum(0)
        dev = None
        if base is not None:
            num = torch.linalg.vector_norm(ys - base, dim=1)
            dev = float((num / (1 + torch.linalg.vector_norm(base, dim=1))).max())
        print(f"{cfg} mode {mode} {which}-blocked nb={nb} ({bs * R * 4 / 1e6:.0f} MB/block): {ms:.3f} ms"
              f"  row_dev vs unblocked {dev}", flush=True)
        del t2, h2, y2, new
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
