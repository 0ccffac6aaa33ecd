"""Synthetic power-law tensors of the FROSTT shapes, on the GPU.

Measurement inputs only (the reference's own generator, generate.py:62-115,
needs ~74 h at these sizes).  Per mode, coordinates follow a truncated
continuous power law on [1, D+1]; draws are deduplicated (set semantics),
topped up until at least M distinct coordinates exist, then down-sampled to
exactly M with a seeded choice; values are U(0,1] as 1 - u; the result is
canonical (identity-sorted, unique).  Deterministic for a given seed, device
type and torch version (torch's Philox CUDA generator).
"""
from __future__ import annotations

import ctypes as C
import math
import os
import time

from . import _native as N
from .coo import CooTensor, canonicalize, unique_coordinates

# BASELINE.json configs[1..4] (exact FROSTT dims), α per mode, seed
CONFIGS = {
    "config1": dict(dims=(1000, 1000, 1000), nnz=100_000, alpha=None, seed=0),
    "nell-2": dict(dims=(12092, 9184, 28818), nnz=76_879_419, alpha=(1.0, 1.0, 1.0), seed=2),
    "flickr-3d": dict(dims=(319686, 28153045, 1607191), nnz=112_890_310, alpha=(1.0, 1.0, 1.0), seed=3),
    "delicious-3d": dict(dims=(532924, 17262471, 2480308), nnz=140_126_181, alpha=(0.3, 1.0, 0.3), seed=4),
    "nell-1": dict(dims=(2902330, 2143368, 25495389), nnz=143_599_552, alpha=(1.0, 1.0, 1.0), seed=5),
}


def _draw_mode(torch, gen, n, dim, alpha):
    u = torch.rand(n, generator=gen, device="cuda", dtype=torch.float64)
    top = float(dim + 1)
    if alpha == 1.0:
        x = torch.exp(u * math.log(top))
    else:
        a = 1.0 - alpha
        x = ((top ** a - 1.0) * u + 1.0) ** (1.0 / a)
    i = torch.floor(x).to(torch.int64) - 1
    return i.clamp_(0, dim - 1).to(torch.int32)


def _coords_of(torch, t: CooTensor):
    idx = torch.empty((t.nnz, t.order), dtype=torch.int32, device="cuda")
    N.call("hbk_coo_export_device", t._dev().ptr, C.c_void_p(idx.data_ptr()), None, None,
           N.stream_ptr())
    return idx


def powerlaw_tensor(dims, nnz: int, alpha, seed: int, scale: float = 1.0) -> CooTensor:
    """Canonical device-resident tensor with per-mode power-law marginals.

    ``scale`` < 1 shrinks nnz (dims unchanged) for quick runs."""
    torch = N.require_device()
    dims = tuple(int(d) for d in dims)
    nnz = int(round(nnz * scale))
    gen = torch.Generator(device="cuda")
    gen.manual_seed(int(seed))
    have = torch.empty((0, len(dims)), dtype=torch.int32, device="cuda")
    need = nnz
    verbose = bool(os.environ.get("HBK_GEN_VERBOSE"))
    for it in range(64):
        tic = time.perf_counter()
        draw = int(math.ceil(1.15 * need)) + 16
        new = torch.stack([_draw_mode(torch, gen, draw, d, a) for d, a in zip(dims, alpha)], dim=1)
        cand = torch.cat([have, new], dim=0)
        zero = torch.zeros(cand.shape[0], dtype=torch.float32, device="cuda")
        uniq = unique_coordinates(CooTensor(dims, cand, zero))
        have = _coords_of(torch, uniq)
        if verbose:
            torch.cuda.synchronize()
            print(f"[gen] iter {it}: drew {draw}, unique {have.shape[0]}/{nnz} "
                  f"({time.perf_counter() - tic:.2f}s)", flush=True)
        if have.shape[0] >= nnz:
            break
        need = nnz - have.shape[0]
    else:
        raise RuntimeError("could not draw enough distinct coordinates")
    if have.shape[0] > nnz:
        keep = torch.randperm(have.shape[0], generator=gen, device="cuda")[:nnz]
        have = have[keep]
    vals = 1.0 - torch.rand(nnz, generator=gen, device="cuda", dtype=torch.float64)
    return canonicalize(CooTensor(dims, have, vals))


def uniform_tensor(dims, nnz: int, seed: int) -> CooTensor:
    """Uniform coordinates (configuration 1 shape), same dedup/down-sample recipe."""
    return powerlaw_tensor(dims, nnz, (0.0,) * len(dims), seed)


def config_tensor(name: str, scale: float = 1.0) -> CooTensor:
    c = CONFIGS[name]
    alpha = c["alpha"] if c["alpha"] is not None else (0.0,) * len(c["dims"])
    return powerlaw_tensor(c["dims"], c["nnz"], alpha, c["seed"], scale=scale)
