"""At-scale parity over whole-slice shards (SURVEY.md §7 hard part 6, §8(c)).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py): used by tests/,
scripts/scale_parity.py and bench.py's cpu_baseline leg as the checker.

Why a shard is an exact check of the full-size build: every output row of
mode n depends only on the nonzeros of its slice, the HB-CSF buckets are
slice-disjoint (formats.py:266-294), split_fibers acts per fiber
(balance.py:65-90) and assign_slice_blocks per slice (balance.py:166-187).
So the arrays the GPU builds for the WHOLE tensor, restricted to a set S of
slices (pointers rebased, schedule units renumbered), must equal bit for bit
what the reference algorithm builds from the nonzeros of S alone — and the
MTTKRP rows of S must agree within the row metric.  The oracle side
(oracle/tenkit_port.py) only ever sees the shard, so it stays within a few
seconds of CPU at benchmark scale, while the GPU side is the full-size build
(wide sort keys, 100M+ nonzeros, u32 pointer ranges).
"""
from __future__ import annotations

import numpy as np

from . import tenkit_port as P


# ------------------------------------------------------------ slice choice
def select_slices(hist: np.ndarray, target_nnz: int, seed: int = 0, runs: int = 6,
                  run_len: int = 48, include_heaviest: bool = True) -> np.ndarray:
    """Row ids of mode-n slices for a parity shard of about ``target_nnz``.

    ``hist[i]`` = nonzeros in slice i of the full tensor.  The shard holds the
    heaviest slice (the B-CSF splitting case; optional), ``runs`` runs of
    ``run_len`` consecutive non-empty slices (light slices side by side,
    bucket boundaries), and a stratified pick over the nnz ranks (every K-th
    slice from heaviest to lightest) filling the rest of the budget, so the
    size distribution of the shard follows the tensor's."""
    hist = np.asarray(hist, dtype=np.int64)
    nz = np.flatnonzero(hist)
    if len(nz) == 0:
        return nz
    rng = np.random.default_rng(seed)
    chosen = set()
    budget = int(target_nnz)
    if include_heaviest:
        top = int(nz[np.argmax(hist[nz])])
        chosen.add(top)
        budget -= int(hist[top])
    for _ in range(runs):
        a = int(rng.integers(0, max(1, len(nz) - run_len)))
        for i in nz[a:a + run_len]:
            if int(i) not in chosen:
                chosen.add(int(i))
                budget -= int(hist[i])
    if budget > 0:
        ranked = nz[np.argsort(-hist[nz], kind="stable")]
        total = int(hist[ranked].sum())
        k = max(1, int(np.ceil(total / max(1, budget))))
        for i in ranked[int(rng.integers(0, k))::k]:
            if budget <= 0:
                break
            if int(i) not in chosen:
                chosen.add(int(i))
                budget -= int(hist[i])
    return np.array(sorted(chosen), dtype=np.int64)


def stratified_slices(hist: np.ndarray, target_nnz: int, seed: int = 0,
                      max_slice_frac: float = 0.25) -> np.ndarray:
    """A CPU-baseline sample: every K-th slice by nnz rank (heaviest to
    lightest), skipping slices heavier than ``max_slice_frac`` of the target
    so no single slice dominates the sample's time."""
    hist = np.asarray(hist, dtype=np.int64)
    nz = np.flatnonzero(hist)
    cap = max(1, int(max_slice_frac * target_nnz))
    nz = nz[hist[nz] <= cap]
    if len(nz) == 0:
        return nz
    ranked = nz[np.argsort(-hist[nz], kind="stable")]
    total = int(hist[ranked].sum())
    k = max(1, int(round(total / max(1, target_nnz))))
    off = int(np.random.default_rng(seed).integers(0, k))
    return np.sort(ranked[off::k])


def member(values, rows) -> np.ndarray:
    """Boolean mask ``values ∈ rows`` through a lookup table (rows are small
    non-negative ids; np.isin would sort 100M+ values)."""
    values = np.asarray(values)
    rows = np.asarray(rows, dtype=np.int64)
    size = int(max(int(values.max(initial=0)), int(rows.max(initial=0)))) + 1
    mark = np.zeros(size, dtype=bool)
    mark[rows] = True
    return mark[values]


def shard_entries(indices: np.ndarray, values: np.ndarray, mode: int, rows: np.ndarray):
    """Nonzeros of the selected slices (rows sorted ascending)."""
    keep = member(indices[:, mode], rows)
    return indices[keep], values[keep]


# ----------------------------------------------------- restriction helpers
def _ranges(ptr: np.ndarray, nodes: np.ndarray):
    """Children of ``nodes`` under pointer array ``ptr`` (concatenated ranges)
    and the rebased pointer array of the selection."""
    ptr = np.asarray(ptr, dtype=np.int64)
    lo = ptr[nodes]
    cnt = ptr[nodes + 1] - lo
    new_ptr = np.concatenate([[0], np.cumsum(cnt)]).astype(np.int64)
    total = int(new_ptr[-1])
    owner = np.repeat(np.arange(len(nodes)), cnt)
    child = (lo[owner] + (np.arange(total) - new_ptr[owner])) if total else np.zeros(0, np.int64)
    return child.astype(np.int64), new_ptr


def restrict_tree(ptrs, idxs, leaf, values, rows):
    """A CSF tree (exported arrays) restricted to the slices whose index is in
    ``rows``; returns (ptrs, idxs, leaf, values, slice_positions)."""
    rows = np.asarray(rows)
    pos = np.flatnonzero(member(idxs[0], rows)).astype(np.int64)
    nodes = pos
    out_ptrs, out_idxs = [], [np.asarray(idxs[0])[pos]]
    for d in range(len(ptrs)):
        child, new_ptr = _ranges(ptrs[d], nodes)
        out_ptrs.append(new_ptr)
        if d + 1 < len(idxs):
            out_idxs.append(np.asarray(idxs[d + 1])[child])
        nodes = child
    return out_ptrs, out_idxs, np.asarray(leaf)[nodes], np.asarray(values)[nodes], pos


def restrict_csl(slice_ptr, slice_idx, rest_idx, values, rows):
    sel = np.flatnonzero(member(slice_idx, rows)).astype(np.int64)
    ent, new_ptr = _ranges(slice_ptr, sel)
    return new_ptr, np.asarray(slice_idx)[sel], np.asarray(rest_idx)[ent], np.asarray(values)[ent]


def restrict_units(units: np.ndarray, mult: np.ndarray, fiber_ptr0: np.ndarray, pos: np.ndarray):
    """Schedule units of the slices at tree positions ``pos``: slice_pos
    renumbered to the shard, fiber ranges rebased, block ids consecutive."""
    units = np.asarray(units, dtype=np.int64).reshape(-1, 4)
    remap = np.full(len(fiber_ptr0) - 1, -1, dtype=np.int64)
    remap[pos] = np.arange(len(pos))
    keep = remap[units[:, 1]] >= 0 if len(units) else np.zeros(0, bool)
    u = units[keep].copy()
    fp = np.asarray(fiber_ptr0, dtype=np.int64)
    new_first = np.concatenate([[0], np.cumsum(fp[pos + 1] - fp[pos])])[:-1]
    shift = fp[u[:, 1]] - new_first[remap[u[:, 1]]]
    u[:, 2] -= shift
    u[:, 3] -= shift
    u[:, 1] = remap[u[:, 1]]
    u[:, 0] = np.arange(len(u))
    return u, np.asarray(mult, dtype=np.int64)[pos]


# ------------------------------------------------------------- OpCounts
def opcount_formula(coo_nnz: int, csl_nnz: int, csf_level_sizes, csf_nnz: int, order: int,
                    rank: int, units: int | None = None):
    """OpCount integers of mttkrp_hbcsf from the structure sizes, as the
    bucket kernels count them (kernels.py:147-151, 222-226, 174-185, 326-342):
    COO and CSL (N-1)·M·R muls, M·R adds; CSF (M + Σ_{d≥1} n_d)·R muls,
    (M + Σ_{1≤d≤N-3} n_d + n_0)·R adds; scheduled CSF (M + Σ_{d≥1} n_d)·R muls,
    (M + Σ_{1≤d≤N-3} n_d + U)·R adds."""
    n = order
    ls = list(csf_level_sizes)
    muls = (n - 1) * (coo_nnz + csl_nnz) + (csf_nnz + sum(ls[1:]) if csf_nnz else 0)
    adds = (coo_nnz + csl_nnz)
    if csf_nnz:
        inner = sum(ls[1:n - 2])
        adds += csf_nnz + inner + (ls[0] if units is None else units)
    return muls * rank, adds * rank


# --------------------------------------------------------------- compare
def compare_hbcsf(gpu: dict, ref: dict, rows) -> dict:
    """gpu: exported full-size arrays {'coo': (idx, val), 'csl': {...},
    'csf': {ptrs, idxs, leaf, values}, 'labels': (slice_idx, labels)};
    ref: oracle dict of the shard (tenkit_port.hbcsf / split_hbcsf).
    Returns {name: bool} per array group (True = bit-exact)."""
    res = {}
    mode = ref["mode_order"][0]
    cidx, cval = gpu["coo"]
    keep = member(cidx[:, mode], rows) if len(cidx) else np.zeros(0, bool)
    res["coo_indices"] = np.array_equal(cidx[keep], ref["coo"][0])
    res["coo_values"] = np.array_equal(cval[keep], ref["coo"][1])
    c = gpu["csl"]
    sp, si, ri, sv = restrict_csl(c["slice_ptr"], c["slice_idx"], c["rest_idx"], c["values"], rows)
    r = ref["csl"]
    res["csl_slice_ptr"] = np.array_equal(sp, r["slice_ptr"])
    res["csl_slice_idx"] = np.array_equal(si, r["slice_idx"])
    res["csl_rest_idx"] = np.array_equal(ri, r["rest_idx"].reshape(ri.shape))
    res["csl_values"] = np.array_equal(sv, r["values"])
    t = gpu["csf"]
    ptrs, idxs, leaf, vals, pos = restrict_tree(t["ptrs"], t["idxs"], t["leaf"], t["values"], rows)
    rt = ref["csf"]
    res["csf_ptrs"] = all(np.array_equal(a, b) for a, b in zip(ptrs, rt["ptrs"])) and len(ptrs) == len(rt["ptrs"])
    res["csf_idxs"] = all(np.array_equal(a, b) for a, b in zip(idxs, rt["idxs"])) and len(idxs) == len(rt["idxs"])
    res["csf_leaf"] = np.array_equal(leaf, rt["leaf"])
    res["csf_values"] = np.array_equal(vals, rt["values"])
    if "labels" in gpu:
        sidx, lab = gpu["labels"]
        sel = member(sidx, rows)
        res["labels"] = np.array_equal(lab[sel], ref["labels"])
    return res


def oracle_shard(indices, values, dims, mode, rows, tau: int = 128, block_size: int = 512):
    """The reference algorithm on the shard: HB-CSF (+labels of the unsplit
    tree), fiber split, block schedule."""
    si, sv = shard_entries(indices, values, mode, rows)
    mo = P.allmode_order(dims, mode)
    h = P.hbcsf(si, sv, dims, mo)  # h["labels"]: classify_slices of the unsplit tree
    hs = P.split_hbcsf(h, tau)
    units, mult = P.block_schedule(hs["csf"], block_size)
    return si, sv, h, hs, units, mult


def gpu_arrays(h, full_csf=None) -> dict:
    """Host copies of a device HB-CSF's arrays (the reference attributes the
    product exports: formats.py field names), plus the slice labels of the
    full unsplit tree when ``full_csf`` (and its labels) are given as
    (slice_idx, labels)."""
    out = {
        "coo": (h.coo_part.indices, h.coo_part.values),
        "csl": {"slice_ptr": h.csl_part.slice_ptr, "slice_idx": h.csl_part.slice_idx,
                "rest_idx": h.csl_part.rest_idx, "values": h.csl_part.values},
        "csf": {"ptrs": h.csf_part.ptrs, "idxs": h.csf_part.idxs, "leaf": h.csf_part.leaf_idx,
                "values": h.csf_part.values},
    }
    if full_csf is not None:
        out["labels"] = full_csf
    return out
