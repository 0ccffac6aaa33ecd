"""Would a communication-aware row partition cut the CP-ALS exchange?
Emulates P ranks on one GPU (like scripts/exchange_volume.py): mode 0 keeps
its nnz-balanced contiguous ranges; every other mode's rows are relabelled so
each row lands in the range of the rank whose shards read it most (then cut
into nnz-balanced contiguous ranges of the relabelled order), optionally
iterated over the modes.  Prints the touched-rows ingress per GPU per sweep
(max / mean over ranks) for the plain and the co-partitioned layout, and the
per-mode nnz imbalance the relabelling costs.

    python scripts/copartition_probe.py nell-1 8 [passes]
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

from paper_1904_03329_b200 import shard
from paper_1904_03329_b200.generate import CONFIGS, config_tensor

R = 32


def ranges_of(counts, P):
    return shard.plan_row_ranges(counts.cpu().numpy(), P)


def owner_map(ranges, dim, dev):
    own = torch.empty(dim, dtype=torch.long, device=dev)
    for r, (lo, hi) in enumerate(ranges):
        own[lo:hi] = r
    return own


def volume(idx, dims, owners, P):
    """Touched-rows ingress (bytes) per rank: rows of factor d read by rank
    r's shards of the other modes and not owned by r."""
    vol = torch.zeros(P, dtype=torch.float64, device=idx.device)
    for d in range(3):
        need = torch.zeros((P, dims[d]), dtype=torch.bool, device=idx.device)
        for n in range(3):
            if n != d:
                need[owners[n][idx[:, n]], idx[:, d]] = True
        need[owners[d], torch.arange(dims[d], device=idx.device)] = False
        vol += need.sum(1).double() * R * 4
    return vol


def main():
    cfg, P = sys.argv[1], int(sys.argv[2])
    passes = int(sys.argv[3]) if len(sys.argv) > 3 else 1
    dims = CONFIGS[cfg]["dims"]
    t = config_tensor(cfg)
    idx = torch.from_numpy(np.ascontiguousarray(t.indices).astype(np.int64)).cuda()
    dev = idx.device
    counts = [torch.bincount(idx[:, d], minlength=dims[d]) for d in range(3)]
    base = [owner_map(ranges_of(counts[d], P), dims[d], dev) for d in range(3)]
    v0 = volume(idx, dims, base, P)
    print(f"{cfg} P={P} contiguous: ingress max {v0.max() / 1e9:.3f} GB mean {v0.mean() / 1e9:.3f} GB",
          flush=True)
    owners = list(base)
    cur = idx.clone()
    for it in range(passes):
        for d in ([1, 2] if it == 0 else [0, 1, 2]):
            # reads of row x of mode d by each rank (through the other modes' shards)
            score = torch.zeros(dims[d] * P, dtype=torch.float64, device=dev)
            for n in range(3):
                if n != d:
                    score += torch.bincount(cur[:, d] * P + owners[n][cur[:, n]], minlength=dims[d] * P).double()
            pref = score.view(dims[d], P).argmax(1)
            # relabel: sort rows by (preferred rank, old id); nnz-balanced cut
            order = torch.argsort(pref * dims[d] + torch.arange(dims[d], device=dev))
            new_id = torch.empty_like(order)
            new_id[order] = torch.arange(dims[d], device=dev)
            cur[:, d] = new_id[cur[:, d]]
            cnt = torch.bincount(cur[:, d], minlength=dims[d])
            rg = ranges_of(cnt, P)
            owners[d] = owner_map(rg, dims[d], dev)
            got = (owners[d][new_id] == pref).float().mean().item()
            print(f"  pass {it} mode {d}: {100 * got:.1f}% of rows owned by their main reader", flush=True)
        v = volume(cur, dims, owners, P)
        imb = []
        for d in range(3):
            per = torch.bincount(owners[d][cur[:, d]], minlength=P).double()
            imb.append(float(per.max() / per.mean()))
        print(f"{cfg} P={P} co-partitioned (pass {it}): ingress max {v.max() / 1e9:.3f} GB mean "
              f"{v.mean() / 1e9:.3f} GB; nnz max/mean per mode {[round(x, 3) for x in imb]}", flush=True)


if __name__ == "__main__":
    main()
