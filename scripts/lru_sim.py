"""Write one mode's factor-row access stream (CSF tree order: each fiber's
leaf rows, then its fiber row; ids: leaf factor rows, then fiber-factor rows
offset by the leaf extent) for scripts/lru_sim.c, then run the LRU
simulation at 126 MB and 63 MB, sequential and interleaved like the kernel.

    python scripts/lru_sim.py nell-1 0
"""
import subprocess
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np

import paper_1904_03329_b200 as hb
from paper_1904_03329_b200.generate import CONFIGS, config_tensor

cfg, mode = sys.argv[1], int(sys.argv[2])
dims = CONFIGS[cfg]["dims"]
t = config_tensor(cfg)
mo = hb.allmode_order(dims, mode)
c = hb.build_csf(t, mo)
fptr = c.ptrs[1].astype(np.int64)
fidx = c.idxs[1].astype(np.int64)
leaf = c.leaf_idx.astype(np.int64)
nF, M = len(fidx), len(leaf)
nC = dims[mo[2]]
# position of each leaf in the stream: its index + number of fibers before it
fib_of = np.repeat(np.arange(nF), np.diff(fptr))
s = np.empty(M + nF, dtype=np.int32)
s[np.arange(M) + fib_of] = leaf
s[fptr[1:] - 1 + np.arange(1, nF + 1)] = nC + fidx
path = "/tmp/stream_%s_%d.bin" % (cfg, mode)
with open(path, "wb") as f:
    np.array([len(s)], dtype=np.int64).tofile(f)
    s.tofile(f)
nrows = nC + dims[mo[1]]
print(f"{cfg} mode {mode}: {M} leaf + {nF} fiber accesses, {nrows} distinct rows possible", flush=True)
subprocess.run(["gcc", "-O2", "-o", "/tmp/lru", str(Path(__file__).parent / "lru_sim.c")], check=True)
for cap_mb in (126, 63):
    cap = int(cap_mb * 1e6 / 128)
    for w, tsz, b in ((1, 1, 1), (14208, 1024, 8)):
        subprocess.run(["/tmp/lru", path, str(nrows), str(cap), str(w), str(tsz), str(b)], check=True)
