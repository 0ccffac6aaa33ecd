"""Multi-GPU partitioner and factor exchange.

Output-mode slices are independent (each output row depends only on its
slice's nonzeros, kernels.py:154-186), so a mode is sharded into contiguous
row ranges balanced by nonzero count; each rank builds the HB-CSF of its
shard and produces its rows with no data-path collective.  Between CP-ALS
modes the updated factor rows are replicated with an all-gather over NCCL
(uneven row counts are padded to the largest shard, one collective).

The range planner is a pure function (unit-tested on CPU); the exchange works
on any torch.distributed backend (gloo tests on CPU, NCCL on the GPUs).
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native as N
from .coo import CooTensor


def plan_row_ranges(slice_nnz, parts: int) -> list[tuple[int, int]]:
    """Split rows [0, len(slice_nnz)) into `parts` contiguous ranges whose
    nonzero counts are as even as whole slices allow: boundary g is the first
    row whose prefix count reaches g*M/parts (lower_bound on the prefix sum)."""
    counts = np.asarray(slice_nnz, dtype=np.int64)
    rows = len(counts)
    if parts < 1:
        raise ValueError("parts must be >= 1")
    prefix = np.concatenate([[0], np.cumsum(counts)])
    total = int(prefix[-1])
    cuts = [0]
    for g in range(1, parts):
        target = (g * total + parts - 1) // parts
        b = int(np.searchsorted(prefix, target, side="left"))
        cuts.append(min(max(b, cuts[-1]), rows))
    cuts.append(rows)
    return [(cuts[g], cuts[g + 1]) for g in range(parts)]


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


def shard_for_rank(t: CooTensor, mode: int, rank: int, world: int):
    """(row range, shard tensor) owned by `rank` for `mode`."""
    ranges = plan_row_ranges(slice_histogram(t, mode).cpu().numpy(), world)
    lo, hi = ranges[rank]
    return (lo, hi), select_rows(t, mode, lo, hi)


def allgather_rows(local, ranges, group=None):
    """Replicate a row-sharded matrix: rank g holds rows ranges[g] of a
    (rows, R) matrix in `local`; returns the full matrix on every rank.  One
    all_gather of max-shard-sized buffers (uneven shards padded)."""
    import torch
    import torch.distributed as dist

    world = len(ranges)
    width = local.shape[1]
    cap = max(hi - lo for lo, hi in ranges)
    buf = torch.zeros((cap, width), dtype=local.dtype, device=local.device)
    buf[: local.shape[0]] = local
    outs = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(outs, buf, group=group)
    full = torch.empty((ranges[-1][1], width), dtype=local.dtype, device=local.device)
    for g, (lo, hi) in enumerate(ranges):
        full[lo:hi] = outs[g][: hi - lo]
    return full
