"""MTTKRP time per mode in fp64 (precision="fp64": the fast kernels on double2
lanes; HBK_F64_GENERIC=1 for the generic kernel) vs
the fp32 fast path, R=32."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

import paper_1904_03329_b200 as hb
from paper_1904_03329_b200.generate import CONFIGS, config_tensor
from paper_1904_03329_b200.kernels import mttkrp_device

cfg = sys.argv[1] if len(sys.argv) > 1 else "nell-2"
dims = CONFIGS[cfg]["dims"]
t = config_tensor(cfg)
f32 = [torch.rand((d, 32), device="cuda") for d in dims]
f64 = [x.double() for x in f32]


def timed(fn, n=5):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n


for mode in range(3):
    h = hb.split_fibers(hb.build_hbcsf(t, hb.allmode_order(dims, mode)), hb.SplitConfig())
    a = timed(lambda: mttkrp_device(h, f32, mode))
    b = timed(lambda: mttkrp_device(h, f64, mode))
    print(f"{cfg} mode {mode}: fp32 fast {a:.3f} ms, fp64 {b:.3f} ms ({b / a:.1f}x)", flush=True)
