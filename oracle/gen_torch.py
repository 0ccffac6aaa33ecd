"""Pure-torch restatement of the benchmark input generator — TEST / BASELINE
INFRASTRUCTURE ONLY.

bench.py's reference arm (``--impl reference``) must run without the
product library, yet time the reference algorithm on the same tensor the
product arm measures.  This module reproduces
``paper_1904_03329_b200.generate.powerlaw_tensor``
with torch operations only: the same torch CUDA Philox draws in the same
order (per mode per top-up round, then ``randperm`` for the down-sample, then
the values), with the product's libhbk dedup / canonicalize replaced by
stable lexicographic torch sorts.  The result is bit-identical (checked by
tests/test_gpu_reference_arm.py); no libhbk symbol is loaded.
"""
from __future__ import annotations

import math

import numpy as np

# BASELINE.json configs (exact FROSTT dims), per-mode α, seed — the same
# table as paper_1904_03329_b200.generate.CONFIGS (tests assert equality)
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


def _lex_perm(torch, x):
    """Stable lexicographic order of the rows of x (column 0 major)."""
    perm = torch.arange(x.shape[0], device=x.device)
    for c in reversed(range(x.shape[1])):
        _, p = torch.sort(x[perm, c], stable=True)
        perm = perm[p]
    return perm


def _unique_rows(torch, x):
    y = x[_lex_perm(torch, x)]
    keep = torch.ones(y.shape[0], dtype=torch.bool, device=y.device)
    if y.shape[0] > 1:
        keep[1:] = (y[1:] != y[:-1]).any(dim=1)
    return y[keep]


def powerlaw_tensor(dims, nnz: int, alpha, seed: int, scale: float = 1.0):
    """(indices int32 (M, N) CUDA, values float64 (M,) CUDA), canonical
    (identity-sorted, unique) — the same tensor as the product generator."""
    import torch

    dims = tuple(int(d) for d in dims)
    nnz = int(round(nnz * scale))
    gen = torch.Generator(device="cuda")
    gen.manual_seed(int(seed))
    have = torch.empty((0, len(dims)), dtype=torch.int32, device="cuda")
    need = nnz
    for _ in range(64):
        draw = int(math.ceil(1.15 * need)) + 16
        new = torch.stack([_draw_mode(torch, gen, draw, d, a) for d, a in zip(dims, alpha)], dim=1)
        have = _unique_rows(torch, torch.cat([have, new], dim=0))
        if have.shape[0] >= nnz:
            break
        need = nnz - have.shape[0]
    else:
        raise RuntimeError("could not draw enough distinct coordinates")
    if have.shape[0] > nnz:
        keep = torch.randperm(have.shape[0], generator=gen, device="cuda")[:nnz]
        have = have[keep]
    vals = 1.0 - torch.rand(nnz, generator=gen, device="cuda", dtype=torch.float64)
    perm = _lex_perm(torch, have)
    return have[perm], vals[perm]


def config_tensor(name: str, scale: float = 1.0):
    c = CONFIGS[name]
    alpha = c["alpha"] if c["alpha"] is not None else (0.0,) * len(c["dims"])
    return powerlaw_tensor(c["dims"], c["nnz"], alpha, c["seed"], scale=scale)


def host_shard(indices, values, mode: int, rows: np.ndarray):
    """Nonzeros of the slices ``rows`` of ``mode`` as host arrays (uint32
    indices, float64 values), selected on the device."""
    import torch

    mark = torch.zeros(int(indices[:, mode].max().item()) + 1 if indices.shape[0] else 1,
                       dtype=torch.bool, device=indices.device)
    r = torch.from_numpy(np.asarray(rows, dtype=np.int64)).to(indices.device)
    mark[r[r < mark.numel()]] = True
    keep = mark[indices[:, mode].long()]
    return (indices[keep].cpu().numpy().view(np.uint32), values[keep].cpu().numpy())


def slice_histogram(indices, mode: int, dim: int) -> np.ndarray:
    import torch

    return torch.bincount(indices[:, mode].long(), minlength=dim).cpu().numpy()
