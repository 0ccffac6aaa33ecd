"""The reference's synthetic-tensor generator and flatten helpers, restated
for tests — TEST INFRASTRUCTURE ONLY.

``generate_raw`` follows ``tenkit.generate.generate_tensor``
(pkg/src/tenkit/generate.py:62-115, helpers :19-59) so that configuration 1
— ``generate_tensor((1000,)*3, 100_000, skew=0.0, seed=0)`` — and the
reference's generator test cases can be reproduced here without the
reference installed.  It must consume numpy's Generator in exactly the
reference's order:
  1. slice counts: one multinomial over Zipf(skew) slice weights
     (generate.py:85-89), capped at the slice capacity, overflow handed to
     the first slices with room (:90-97);
  2. per non-empty slice, in slice order, ``count`` distinct mixed-radix
     codes over the remaining modes (first remaining mode fastest):
     near-full slices are a permutation prefix (:33-39); otherwise rounds of
     2x-oversampled draws — Zipf(skew) first coordinate for 12 rounds, then
     uniform — each round keeping the first occurrence of every code
     (:40-59);
  3. values ``1 - rng.random(M)`` (:114).
Not part of the product: the benchmark inputs (configs 2-5) come from the
Appendix-A generator (paper_1904_03329_b200.generate), because this one
costs ~74 h at FROSTT sizes.
"""
from __future__ import annotations

import math

import numpy as np


class CapacityError(ValueError):
    """coo.py:31-32 (the reference raises its CapacityError here)."""


def zipf_weights(n: int, skew: float) -> np.ndarray:
    w = np.arange(1, n + 1, dtype=np.float64) ** (-skew)
    return w / w.sum()


def distinct_codes(rng, radices, count: int, skew: float) -> np.ndarray:
    cells = math.prod(radices)
    if count > cells:
        raise ValueError("slice cannot hold that many nonzeros")
    if count > cells // 2:
        if cells > 20_000_000:
            raise CapacityError(f"refusing to enumerate {cells} cells to fill a near-complete slice")
        return rng.permutation(cells)[:count].astype(np.int64)
    weights = zipf_weights(radices[0], skew)
    kept = np.zeros(0, dtype=np.int64)
    rnd = 0
    while kept.size < count:
        n = max(2 * (count - kept.size), 256)
        if rnd < 12:
            lead = rng.choice(radices[0], size=n, p=weights)
        else:
            lead = rng.integers(0, radices[0], size=n)
        code = lead.astype(np.int64)
        stride = radices[0]
        for r in radices[1:]:
            code += rng.integers(0, r, size=n).astype(np.int64) * stride
            stride *= r
        pool = np.concatenate([kept, code])
        _, first = np.unique(pool, return_index=True)
        kept = pool[np.sort(first)]
        rnd += 1
    return kept[:count]


def generate_raw(dims, nnz: int, skew: float = 1.0, seed: int = 0):
    """(dims, indices int64 (M, N), values float64 (M,)) before canonicalisation."""
    dims = tuple(int(d) for d in dims)
    if len(dims) < 3:
        raise ValueError("tensor order must be >= 3")
    if skew < 0:
        raise ValueError("skew must be nonnegative")
    total = math.prod(dims)
    if nnz < 0 or nnz > total:
        raise ValueError(f"nnz must lie in [0, {total}], got {nnz}")
    rng = np.random.default_rng(seed)
    radices = dims[1:]
    room = math.prod(radices)
    counts = np.minimum(rng.multinomial(nnz, zipf_weights(dims[0], skew)), room)
    left = nnz - int(counts.sum())
    i = 0
    while left > 0 and i < dims[0]:
        extra = min(room - int(counts[i]), left)
        counts[i] += extra
        left -= extra
        i += 1
    lead_col, code_parts = [], []
    for s, c in enumerate(counts.tolist()):
        if c:
            code_parts.append(distinct_codes(rng, radices, int(c), skew))
            lead_col.append(np.full(int(c), s, dtype=np.int64))
    cols = [np.concatenate(lead_col) if lead_col else np.zeros(0, dtype=np.int64)]
    code = np.concatenate(code_parts) if code_parts else np.zeros(0, dtype=np.int64)
    for r in radices:
        code, digit = np.divmod(code, r)
        cols.append(digit)
    idx = np.stack(cols, axis=1)
    return dims, idx, 1.0 - rng.random(idx.shape[0])


def flatten_csf(tree: dict):
    """formats.py:171-191 on an oracle tree dict: (indices (M, N) uint32 in
    tree order, values)."""
    mo = tree["mode_order"]
    n = len(mo)
    m = len(tree["values"])
    perm = np.empty((m, n), dtype=np.uint32)
    perm[:, n - 1] = tree["leaf"]
    off = np.asarray(tree["ptrs"][n - 2])
    perm[:, n - 2] = np.repeat(tree["idxs"][n - 2], np.diff(off))
    for d in range(n - 3, -1, -1):
        off = off[np.asarray(tree["ptrs"][d])]
        perm[:, d] = np.repeat(tree["idxs"][d], np.diff(off))
    out = np.empty_like(perm)
    out[:, list(mo)] = perm
    return out, tree["values"]
