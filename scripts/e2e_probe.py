"""Host<->device transfer variants for the host-array MTTKRP calling
convention (nell-2 factor sizes).  Run on the GPU box."""
import time
import numpy as np
import torch

dims = (12092, 9184, 28818)
R = 32
rng = np.random.default_rng(0)
f64 = [rng.random((d, R)) for d in dims]
torch.cuda.init()
dev = [torch.empty((d, R), dtype=torch.float32, device="cuda") for d in dims]


def t(fn, reps=20):
    fn(); torch.cuda.synchronize()
    tic = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - tic) / reps * 1e3


print("isfinite all 3      %.3f ms" % t(lambda: [np.isfinite(f).all() for f in f64]))
print("astype f32 (3)      %.3f ms" % t(lambda: [np.ascontiguousarray(f, np.float32) for f in f64]))
print("astype+cuda (3)     %.3f ms" % t(lambda: [torch.from_numpy(np.ascontiguousarray(f, np.float32)).cuda() for f in f64]))
pin32 = [torch.empty((d, R), dtype=torch.float32, pin_memory=True) for d in dims]
pin64 = [torch.empty((d, R), dtype=torch.float64, pin_memory=True) for d in dims]


def pinned32():
    for f, p, d in zip(f64, pin32, dev):
        np.copyto(p.numpy(), f, casting="same_kind")
        d.copy_(p, non_blocking=True)


def pinned64():
    for f, p, d in zip(f64, pin64, dev):
        np.copyto(p.numpy(), f)
        d.copy_(p.cuda(non_blocking=True))


print("pinned f32 stage    %.3f ms" % t(pinned32))
print("pinned f64 stage    %.3f ms" % t(pinned64))
print("copyto f64->f32 only %.3f ms" % t(lambda: [np.copyto(p.numpy(), f, casting="same_kind") for f, p in zip(f64, pin32)]))
print("H2D pinned f32 only %.3f ms" % t(lambda: [d.copy_(p, non_blocking=True) for d, p in zip(dev, pin32)]))
y = torch.rand((28818, R), device="cuda")
print("y.double().cpu().numpy() %.3f ms" % t(lambda: y.double().cpu().numpy()))
ypin = torch.empty((28818, R), dtype=torch.float64, pin_memory=True)


def pinned_out():
    ypin.copy_(y.double(), non_blocking=True)
    torch.cuda.current_stream().synchronize()
    return ypin.numpy().copy()


print("pinned out + copy   %.3f ms" % t(pinned_out))


def pinned_out32():
    p = pin32[2]
    p.copy_(y, non_blocking=True)
    torch.cuda.current_stream().synchronize()
    return p.numpy().astype(np.float64)


print("pinned out f32+astype %.3f ms" % t(pinned_out32))
