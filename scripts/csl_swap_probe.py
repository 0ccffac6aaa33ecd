"""How many rows would the CSL part gather if its singleton-fiber slices were
walked as CSF under the swapped order (mode, rest[1], rest[0])?  CSL: 2 rows
per nonzero; swapped CSF: 1 per nonzero + 1 per distinct (slice, rest[1])."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np

import paper_1904_03329_b200 as hb
from paper_1904_03329_b200.generate import CONFIGS, config_tensor

cfg = sys.argv[1] if len(sys.argv) > 1 else "delicious-3d"
dims = CONFIGS[cfg]["dims"]
t = config_tensor(cfg, scale=float(sys.argv[2]) if len(sys.argv) > 2 else 1.0)
for mode in range(3):
    mo = hb.allmode_order(dims, mode)
    h = hb.build_hbcsf(t, mo)
    s = h.csl_part
    if s.nnz == 0:
        print(cfg, mode, "no CSL")
        continue
    idx = np.empty((s.nnz, 3), dtype=np.uint32)
    idx[:, mo[0]] = np.repeat(s.slice_idx, np.diff(s.slice_ptr))
    idx[:, list(mo[1:])] = s.rest_idx
    c = hb.build_csf(hb.CooTensor(dims, idx, s.values), (mo[0], mo[2], mo[1]))
    rows_csl = 2 * s.nnz
    rows_swap = s.nnz + c.num_fibers
    print(f"{cfg} mode {mode}: CSL nnz {s.nnz} slices {s.num_slices}; swapped fibers {c.num_fibers}; "
          f"rows {rows_csl} -> {rows_swap} ({rows_swap / rows_csl:.2f}x)", flush=True)
