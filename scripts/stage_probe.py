"""hbk_stage_f64_to_f32 alone: narrowing + chunked H2D of nell-2's mode-0
factors (9184 x 32 and 28818 x 32 float64), wall time per call (synchronised)."""
import ctypes as C
import statistics
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

from paper_1904_03329_b200 import _native as N

N.load_library()
rng = np.random.default_rng(0)
rows = [int(r) for r in (sys.argv[1].split(",") if len(sys.argv) > 1 else (9184, 28818))]
src = [rng.random((r, 32)) for r in rows]
stage = [torch.empty((r, 32), dtype=torch.float32, pin_memory=True) for r in rows]
dev = [torch.empty((r, 32), dtype=torch.float32, device="cuda") for r in rows]
k = len(rows)
flags = (C.c_int32 * k)()
args = ((C.c_void_p * k)(*[s.ctypes.data for s in src]), (C.c_int64 * k)(*[s.size for s in src]), k,
        (C.c_void_p * k)(*[s.data_ptr() for s in stage]), (C.c_void_p * k)(*[d.data_ptr() for d in dev]),
        flags)
ts, ti = [], []
for it in range(40):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    N.call("hbk_stage_f64_to_f32", *args, N.stream_ptr())
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    ti.append(t1 - t0)
    ts.append(t2 - t0)
assert np.array_equal(dev[-1].cpu().numpy(), src[-1].astype(np.float32))
print(f"rows {rows}: issue {statistics.median(ti[5:]) * 1e3:.3f} ms, synced {statistics.median(ts[5:]) * 1e3:.3f} ms",
      flush=True)
