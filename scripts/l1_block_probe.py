"""Would L1-sized leaf blocking of the LONG fibers speed up the L2-resident
configurations (nell-2)?  The nell-2 kernel is bound by L2 -> SM throughput
at a 26% L1 hit rate; the long fibers (30% of the nonzeros sit in fibers
> 128) sweep the leaf rows and evict the Zipf head (profiles/r2_nell2_ceiling.md).

Emulation with the existing kernels: the nonzeros of fibers longer than T are
cut out into their own tensor whose slice index is remapped block-major by
the leaf index, i' = (k // BB) * dims[mode] + i, so the persistent kernel
walks that tensor leaf-block by leaf-block and every SM's L1 holds the
current block's BB leaf rows; the short-fiber rest runs as a second tensor
(its L1 no longer swept).  Times t(short) + t(long, blocked) against
t(full) and checks the summed rows.

  python scripts/l1_block_probe.py nell-2 0 128,512 768,1536,3072
"""
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import ctypes as C

import torch

import paper_1904_03329_b200 as hb
from paper_1904_03329_b200 import _native as N
from paper_1904_03329_b200.generate import CONFIGS, config_tensor
from paper_1904_03329_b200.kernels import mttkrp_device

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


def build(dims, idx, vals, mo):
    t = hb.canonicalize(hb.CooTensor(tuple(dims), idx, vals))
    return hb.split_fibers(hb.build_hbcsf(t, mo), hb.SplitConfig())


def main():
    cfg, mode = sys.argv[1], int(sys.argv[2])
    Ts = [int(x) for x in sys.argv[3].split(",")]
    BBs = [int(x) for x in sys.argv[4].split(",")]
    dims = CONFIGS[cfg]["dims"]
    t = config_tensor(cfg)
    idx = torch.empty((t.nnz, 3), dtype=torch.int32, device="cuda")
    vals = torch.empty(t.nnz, dtype=torch.float64, device="cuda")
    N.call("hbk_coo_export_device", t._dev().ptr, C.c_void_p(idx.data_ptr()),
           C.c_void_p(vals.data_ptr()), None, N.stream_ptr())
    mo = hb.allmode_order(dims, mode)
    g = torch.Generator(device="cuda").manual_seed(1)
    f = [torch.rand((d, R), device="cuda", generator=g) for d in dims]
    h = hb.split_fibers(hb.build_hbcsf(t, mo), hb.SplitConfig())
    base_ms, y = timed(h, f, mode)
    base = y.double()
    del h, y
    print(f"{cfg} mode {mode} leaf dim {dims[mo[2]]}: full {base_ms:.3f} ms", flush=True)
    key = idx[:, mo[0]].long() * dims[mo[1]] + idx[:, mo[1]].long()
    _, inv, cnt = torch.unique(key, return_inverse=True, return_counts=True)
    flen = cnt[inv]
    del key, inv, cnt
    for T in Ts:
        long_m = flen > T
        nl = int(long_m.sum())
        si, sv = idx[~long_m].contiguous(), vals[~long_m].contiguous()
        li, lv = idx[long_m].contiguous(), vals[long_m].contiguous()
        hs = build(dims, si, sv, mo)
        s_ms, ys = timed(hs, f, mode)
        del hs
        print(f"  T={T}: long-fiber nnz {nl} ({nl / t.nnz:.1%}); short part {s_ms:.3f} ms", flush=True)
        hl = build(dims, li, lv, mo)
        l_ms, yl = timed(hl, f, mode)
        del hl
        print(f"    long part unblocked {l_ms:.3f} ms -> sum {s_ms + l_ms:.3f} ms", flush=True)
        for BB in BBs:
            nb = (dims[mo[2]] + BB - 1) // BB
            new = li.clone()
            new[:, mode] = (li[:, mo[2]] // BB) * dims[mode] + li[:, mode]
            d2 = list(dims)
            d2[mode] = nb * dims[mode]
            hb2 = build(d2, new, lv, mo)
            f2 = list(f)
            f2[mode] = torch.empty((d2[mode], R), device="cuda")
            b_ms, yb = timed(hb2, f2, mode)
            ysum = ys.double() + yb.view(nb, dims[mode], R).double().sum(0)
            num = torch.linalg.vector_norm(ysum - base, dim=1)
            dev = float((num / (1 + torch.linalg.vector_norm(base, dim=1))).max())
            print(f"    long part blocked BB={BB} ({BB * R * 4 / 1024:.0f} KB, {nb} blocks): {b_ms:.3f} ms"
                  f" -> sum {s_ms + b_ms:.3f} ms vs full {base_ms:.3f}  row_dev {dev:.2e}", flush=True)
            del hb2, yb, new
            torch.cuda.empty_cache()
        del ys, yl, si, sv, li, lv


if __name__ == "__main__":
    main()
