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
    import os, time
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


# ------------------------------------------------------------------------
# The reference's own generator (generate.py:62-115), restated so that
# config 1 — tenkit.generate_tensor((1000,)*3, 100_000, skew=0.0, seed=0) —
# can be produced here bit for bit.  It consumes numpy's Generator in the
# same order as the reference (multinomial slice counts, then per slice a
# Zipf-weighted first coordinate and uniform rest, de-duplicated keeping the
# first occurrence), so the tensor is identical for a given seed.  A host
# input generator, not part of the kernel path; the result is canonicalised
# on the GPU.
def _powers(n: int, skew: float):
    import numpy as np

    w = np.arange(1, n + 1, dtype=np.float64) ** (-skew)
    return w / w.sum()


def _slice_codes(rng, sub, count: int, skew: float):
    """``count`` distinct mixed-radix codes over ``sub`` (first mode fastest),
    first coordinate Zipf(skew)-weighted (generate.py:25-59)."""
    import numpy as np

    from .coo import CapacityError

    cap = math.prod(sub)
    if count > cap:
        raise ValueError("slice cannot hold that many nonzeros")
    if count > cap // 2:
        if cap > 20_000_000:
            raise CapacityError(f"refusing to enumerate {cap} cells to fill a near-complete slice")
        return rng.permutation(cap)[:count].astype(np.int64)
    p = _powers(sub[0], skew)
    have = np.empty(0, dtype=np.int64)
    rounds = 0
    while have.size < count:
        draw = max(2 * (count - have.size), 256)
        lead = (rng.choice(sub[0], size=draw, p=p) if rounds < 12
                else rng.integers(0, sub[0], size=draw)).astype(np.int64)
        code, radix = lead, sub[0]
        for d in sub[1:]:
            code = code + rng.integers(0, d, size=draw).astype(np.int64) * radix
            radix *= d
        pool = np.concatenate([have, code])
        _, first = np.unique(pool, return_index=True)
        have = pool[np.sort(first)]
        rounds += 1
    return have[:count]


def _generate_raw(dims, nnz: int, skew: float, seed: int):
    """Coordinates and values before canonicalisation (generate.py:76-114)."""
    import numpy as np

    dims = tuple(int(d) for d in dims)
    if len(dims) < 3:
        raise ValueError("tensor order must be >= 3")
    if skew < 0:
        raise ValueError("skew must be nonnegative")
    cells = math.prod(dims)
    if not 0 <= nnz <= cells:
        raise ValueError(f"nnz must lie in [0, {cells}], got {nnz}")
    rng = np.random.default_rng(seed)
    sub = dims[1:]
    room = math.prod(sub)
    per_slice = np.minimum(rng.multinomial(nnz, _powers(dims[0], skew)), room)
    spill = nnz - int(per_slice.sum())
    for i in range(dims[0]):  # overflow goes to the first slices with room
        if spill <= 0:
            break
        add = min(room - int(per_slice[i]), spill)
        per_slice[i] += add
        spill -= add
    rows, codes = [], []
    for i, c in enumerate(per_slice.tolist()):
        if c:
            codes.append(_slice_codes(rng, sub, int(c), skew))
            rows.append(np.full(int(c), i, dtype=np.int64))
    cols = [np.concatenate(rows)] if rows else [np.zeros(0, dtype=np.int64)]
    code = np.concatenate(codes) if codes else np.zeros(0, dtype=np.int64)
    for d in sub:
        cols.append(code % d)
        code = code // d
    idx = np.stack(cols, axis=1)
    vals = 1.0 - rng.random(idx.shape[0])
    return dims, idx, vals


def generate_tensor(dims, nnz: int, skew: float = 1.0, seed: int = 0) -> CooTensor:
    """Canonical random tensor with Zipf(skew) slice and second-mode skew,
    uniform values in (0, 1] (generate.py:62-115; same result per seed)."""
    dims, idx, vals = _generate_raw(dims, nnz, skew, seed)
    return canonicalize(CooTensor(dims, idx, vals))
