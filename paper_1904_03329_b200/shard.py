"""Multi-GPU row partitioner.

Output-mode slices are independent (each output row depends only on its
slice's nonzeros, kernels.py:154-186), so a mode is sharded into contiguous
row ranges; each rank builds the HB-CSF of its shard and produces its rows
with no data-path collective.  The ranges balance a cost, not the nonzero
count: a slice costs its gathered factor rows (nonzeros + fibers) plus
ROW_COST per output row (empty rows included).  Balancing nonzeros alone left
the rank holding the long tail of light and empty slices 2-3x slower than the
others at 8 ranks (nell-1 mode 2: 22.1M of 25.5M rows on the last rank); the
per-rank timings behind ROW_COST are in scripts/shard_scaling.py's log
(profiles/r2s3/shard_scaling*.log).  The exchanges of the row-sharded CP-ALS
live in distributed.py.

The range planner is a pure function (unit-tested on CPU).
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native as N
from .coo import CooTensor, allmode_order

# gathered-row equivalents per output row: least-squares fit of per-rank MTTKRP
# times (configs 2-5, 2/4/8 ranks) to gathered rows and output rows gives
# 0.0095-0.0117 ms per M gathered rows and 0.024-0.085 ms per M rows
ROW_COST = 4


def plan_row_ranges(slice_nnz, parts: int) -> list[tuple[int, int]]:
    """Split rows [0, len(slice_nnz)) into `parts` contiguous ranges whose
    weights (nonzero counts, partition_costs, or calibrated float weights) are
    as even as whole slices allow: boundary g is the first row whose prefix
    weight reaches g*M/parts (lower_bound on the prefix sum)."""
    w = np.asarray(slice_nnz)
    integral = np.issubdtype(w.dtype, np.integer)
    w = w.astype(np.int64 if integral else np.float64)
    rows = len(w)
    if parts < 1:
        raise ValueError("parts must be >= 1")
    prefix = np.concatenate([[0], np.cumsum(w)])
    total = prefix[-1]
    cuts = [0]
    for g in range(1, parts):
        target = (g * int(total) + parts - 1) // parts if integral else g * float(total) / parts
        b = int(np.searchsorted(prefix, target, side="left"))
        cuts.append(min(max(b, cuts[-1]), rows))
    cuts.append(rows)
    return [(cuts[g], cuts[g + 1]) for g in range(parts)]


def refine_row_ranges(costs, ranges, times) -> list[tuple[int, int]]:
    """One calibration pass over a first partition: every row of range r is
    re-weighted by times[r] / cost(range r) — the measured time per cost unit
    of the rank that ran it — and the rows are cut again.  Corrects what the
    static cost model misses (per-bucket and per-locality rates differ by
    configuration: 15% rms error of the best global fit)."""
    c = np.asarray(costs, dtype=np.float64)
    w = c.copy()
    rates = []
    for (lo, hi), t in zip(ranges, times):
        tot = float(c[lo:hi].sum())
        rates.append(t / tot if tot > 0 and t > 0 else None)
    known = [r for r in rates if r is not None]
    fallback = float(np.mean(known)) if known else 1.0
    for (lo, hi), r in zip(ranges, rates):
        w[lo:hi] *= r if r is not None else fallback
    return plan_row_ranges(w, len(ranges))


def partition_costs(t: CooTensor, mode: int):
    """Per-row cost of a mode's slices for plan_row_ranges: nonzeros + fibers
    of the CSF tree in allmode_order (the factor rows the MTTKRP gathers for
    the slice) + ROW_COST, on the device (int64 CUDA tensor)."""
    mid = allmode_order(t.dims, mode)[1]
    return slice_histogram(t, mode) + fiber_histogram(t, mode, mid) + ROW_COST


def fiber_histogram(t: CooTensor, mode: int, mid_mode: int):
    """Fibers per mode-``mode`` slice of the tree ordered (mode, mid_mode, ...):
    distinct (mode, mid_mode) coordinate pairs, counted on the device."""
    torch = N.require_device()
    hist = torch.empty(t.dims[mode], dtype=torch.int64, device="cuda")
    N.call("hbk_coo_fiber_histogram", t._dev().ptr, int(mode), int(mid_mode),
           C.c_void_p(hist.data_ptr()), N.stream_ptr())
    return hist


def slice_histogram(t: CooTensor, mode: int):
    """Nonzeros per mode-``mode`` slice, counted on the device (int64 CUDA tensor)."""
    torch = N.require_device()
    hist = torch.empty(t.dims[mode], dtype=torch.int64, device="cuda")
    N.call("hbk_coo_slice_histogram", t._dev().ptr, int(mode), C.c_void_p(hist.data_ptr()),
           N.stream_ptr())
    return hist


def select_rows(t: CooTensor, mode: int, lo: int, hi: int) -> CooTensor:
    """Entries whose mode-``mode`` coordinate lies in [lo, hi), on the device."""
    out = N.new_out()
    N.call("hbk_coo_select_rows", t._dev().ptr, int(mode), int(lo), int(hi), N.stream_ptr(),
           C.byref(out))
    return CooTensor._from_handle(N.Handle(out, "hbk_coo_release"))


def shard_rows(t: CooTensor, mode: int, lo: int, hi: int) -> CooTensor:
    """Entries whose mode-``mode`` coordinate lies in [lo, hi), rebased: the
    shard has dims[mode] = hi - lo and coordinates shifted by -lo, so its
    MTTKRP produces exactly rows [lo, hi) of the full output."""
    out = N.new_out()
    N.call("hbk_coo_shard_rows", t._dev().ptr, int(mode), int(lo), int(hi), N.stream_ptr(),
           C.byref(out))
    return CooTensor._from_handle(N.Handle(out, "hbk_coo_release"))
