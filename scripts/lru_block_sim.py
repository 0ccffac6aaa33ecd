"""Would leaf-blocking the heavy slices cut the HBM-resident traffic?  LRU
replay (scripts/lru_sim.c) of one mode's factor-row stream in tree order vs
an order in which the slices with >= MIN nonzeros are processed leaf-block
by leaf-block (block = BLOCK_MB of leaf rows): per block, each heavy slice's
fibers restricted to the block (leaf rows, then the fiber row), plus one
access to the slice's output row (its partial-row add); the other slices
follow in tree order.

    python scripts/lru_block_sim.py nell-1 0 [BLOCK_MB] [MIN] [ORDER]
ORDER: "ref" (allmode_order) or "swap" (the two non-target modes swapped).
"""
import subprocess
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np

import paper_1904_03329_b200 as hb
from paper_1904_03329_b200.generate import CONFIGS, config_tensor

cfg, mode = sys.argv[1], int(sys.argv[2])
block_mb = float(sys.argv[3]) if len(sys.argv) > 3 else 24.0
min_nnz = int(sys.argv[4]) if len(sys.argv) > 4 else 2048
order = sys.argv[5] if len(sys.argv) > 5 else "ref"
dims = CONFIGS[cfg]["dims"]
t = config_tensor(cfg)
mo = hb.allmode_order(dims, mode)
if order == "swap":
    mo = (mo[0], mo[2], mo[1])
c = hb.build_csf(t, mo)
sptr = c.ptrs[0].astype(np.int64)
fptr = c.ptrs[1].astype(np.int64)
fidx = c.idxs[1].astype(np.int64)
leaf = c.leaf_idx.astype(np.int64)
S, nF, M = len(sptr) - 1, len(fidx), len(leaf)
nC, nB = dims[mo[2]], dims[mo[1]]
BB = max(1, int(block_mb * 1e6 / 128))
fib_slice = np.repeat(np.arange(S), np.diff(sptr))
nz_fib = np.repeat(np.arange(nF), np.diff(fptr))
nz_slice = fib_slice[nz_fib]
slice_nnz = np.diff(fptr[sptr])
heavy = slice_nnz >= min_nnz
print(f"{cfg} mode {mode} order {mo}: {M} nnz, {nF} fibers, {S} slices; {heavy.sum()} slices >= {min_nnz} "
      f"hold {slice_nnz[heavy].sum()} nnz; leaf blocks of {BB} rows ({(nC + BB - 1) // BB} blocks)", flush=True)


def tree_stream(sel):
    """factor-row ids of the nonzeros/fibers of the selected nonzeros, tree order"""
    nz = np.nonzero(sel)[0]
    f = nz_fib[nz]
    last = np.ones(len(nz), bool)
    last[:-1] = f[1:] != f[:-1]
    n_out = len(nz) + last.sum()
    out = np.empty(n_out, np.int64)
    pos = np.arange(len(nz)) + np.concatenate([[0], np.cumsum(last)[:-1]])
    out[pos] = leaf[nz]
    out[pos[last] + 1] = nC + fidx[f[last]]
    return out


hz = heavy[nz_slice]
# blocked part: sort heavy nonzeros by (block, slice, fiber) (stable keeps leaf order)
nzh = np.nonzero(hz)[0]
blk = leaf[nzh] // BB
o = np.lexsort((nzh, nz_slice[nzh], blk))
nzh = nzh[o]
blk = blk[o]
sl = nz_slice[nzh]
f = nz_fib[nzh]
lastf = np.ones(len(nzh), bool)
lastf[:-1] = (f[1:] != f[:-1]) | (blk[1:] != blk[:-1])
lasts = np.ones(len(nzh), bool)
lasts[:-1] = (sl[1:] != sl[:-1]) | (blk[1:] != blk[:-1])
n_out = len(nzh) + lastf.sum() + lasts.sum()
bs = np.empty(n_out, np.int64)
extra = np.cumsum(lastf.astype(np.int64) + lasts.astype(np.int64))
pos = np.arange(len(nzh)) + np.concatenate([[0], extra[:-1]])
bs[pos] = leaf[nzh]
bs[pos[lastf] + 1] = nC + fidx[f[lastf]]
bs[pos[lasts] + 1 + lastf[lasts]] = nC + nB + c.idxs[0].astype(np.int64)[sl[lasts]]  # output row
streams = {"tree": tree_stream(np.ones(M, bool)),
           "blocked": np.concatenate([bs, tree_stream(~hz)])}
nrows = nC + nB + dims[mode]
subprocess.run(["gcc", "-O2", "-o", "/tmp/lru", str(Path(__file__).parent / "lru_sim.c")], check=True)
for name, s in streams.items():
    path = f"/tmp/stream_{cfg}_{mode}_{name}.bin"
    with open(path, "wb") as fh:
        np.array([len(s)], dtype=np.int64).tofile(fh)
        s.astype(np.int32).tofile(fh)
    print(f"{name}: {len(s)} accesses", flush=True)
    for cap_mb in (126, 63):
        subprocess.run(["/tmp/lru", path, str(nrows), str(int(cap_mb * 1e6 / 128)), "1", "1", "1"], check=True)
