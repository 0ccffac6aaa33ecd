"""hbk_als_update alone: time and effective bandwidth at nell-1 row counts."""
import ctypes as C
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

from paper_1904_03329_b200 import _native as N

N.require_device()
for rows in (2_902_330, 2_143_368, 25_495_389):
    Y = torch.rand((rows, 32), device="cuda")
    F = torch.empty_like(Y)
    M = torch.rand((32, 32), device="cuda")
    w = torch.rand(32, device="cuda")
    G = torch.empty((32, 32), dtype=torch.float64, device="cuda")
    inner = torch.empty(1, dtype=torch.float64, device="cuda")
    args = lambda inn: (C.c_void_p(Y.data_ptr()), rows, 32, C.c_void_p(M.data_ptr()), C.c_void_p(w.data_ptr()),
                        C.c_void_p(F.data_ptr()), C.c_void_p(G.data_ptr()), inn, N.stream_ptr())
    for inn in (None, C.c_void_p(inner.data_ptr())):
        N.call("hbk_als_update", *args(inn))
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(10):
            N.call("hbk_als_update", *args(inn))
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / 10
        print(f"rows {rows:>10d} inner={inn is not None}: {ms:.3f} ms  {rows * 256 / ms / 1e6:.0f} GB/s", flush=True)
    del Y, F
