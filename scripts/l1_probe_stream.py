"""Write the nell-2 mode-m row-access stream in the MTTKRP's order (slices in
tree order; per fiber its leaf rows, then the fiber's B row — the
B-position stream), with row ids relabelled by access frequency (0 = hottest;
C and B rows share one id space), for scripts/l1_probe.cu.

    python scripts/l1_probe_stream.py nell-2 0 /tmp/stream.bin
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np

import paper_1904_03329_b200 as hb
from paper_1904_03329_b200.generate import CONFIGS, config_tensor

cfg, mode, out = sys.argv[1], int(sys.argv[2]), sys.argv[3]
# optional: flag (bit 31) the leaf positions of fibers longer than SCAN so the
# probe can load them with an L1 evict-first / no-allocate hint
scan = int(sys.argv[4]) if len(sys.argv) > 4 else 0
# optional: "reorder" — all positions of fibers <= SCAN first (tree order),
# then the long fibers' positions (a two-phase plan: the short-fiber work runs
# together, the sweeps after it)
reorder = len(sys.argv) > 5 and sys.argv[5] == "reorder"
dims = CONFIGS[cfg]["dims"]
t = config_tensor(cfg)
mo = hb.allmode_order(dims, mode)
c = hb.build_csf(t, mo)
lp = c.ptrs[1]
leaf = c.leaf_idx.astype(np.int64)
fj = c.idxs[1].astype(np.int64) + dims[mo[2]]  # B rows after the C rows
F = len(fj)
fs = np.diff(lp)
# position of each fiber's B entry: after its leaves
n = len(leaf) + F
ids = np.empty(n, dtype=np.int64)
bpos = lp[1:] + np.arange(1, F + 1) - 1          # index of the B slot of fiber f
mask = np.ones(n, bool)
mask[bpos] = False
ids[mask] = leaf
ids[bpos] = fj
vals = np.random.default_rng(0).random(n).astype(np.float32)
cnt = np.bincount(ids, minlength=dims[mo[1]] + dims[mo[2]])
rank = np.empty_like(cnt)
rank[np.argsort(-cnt, kind="stable")] = np.arange(len(cnt))
pairs = np.empty((n, 2), dtype=np.uint32)
pairs[:, 0] = rank[ids]
if scan:
    long_f = np.repeat(fs > scan, fs)          # per leaf position, in leaf order
    flag = np.zeros(n, bool)
    flag[mask] = long_f
    flag[bpos] = fs > scan                      # the fiber's B row goes with it
    if reorder:
        pairs = np.concatenate([pairs[~flag], pairs[flag]])
        print(f"reordered: {int((~flag).sum())} short-fiber positions first, {int(flag.sum())} after")
    else:
        pairs[flag, 0] |= np.uint32(1 << 31)
    print(f"flagged {flag.mean():.3f} of accesses (fibers > {scan})")
pairs[:, 1] = vals.view(np.uint32)
with open(out, "wb") as fp:
    np.array([n, len(cnt)], dtype=np.uint32).tofile(fp)
    pairs.tofile(fp)
top = np.cumsum(np.sort(cnt)[::-1]) / n
print(f"{cfg} mode {mode}: {n} row accesses, {len(cnt)} rows; top 512/1024/1536 rows cover "
      f"{top[511]:.3f}/{top[1023]:.3f}/{top[1535]:.3f}")
