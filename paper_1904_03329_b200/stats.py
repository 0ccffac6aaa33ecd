"""Slice/fiber population statistics (coo.py:250-325).

``compute_stats`` mirrors the reference's TensorStats: the tensor is sorted
and compressed under the mode order by libhbk's CSF builder on the GPU (K1,
K2), and the statistics are device reductions over its pointer arrays
(hbk_csf_population) — the reference's group counting (coo.py:304-311)
without a host sort or an export.
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Sequence

from .coo import CooTensor, _check_mode_order
from .formats import build_csf, mean_std, population


@dataclass(frozen=True)
class TensorStats:
    """Slice/fiber nonzero statistics under a mode order (coo.py:250-278).
    Standard deviations are population (divide by count)."""

    order: int
    dims: tuple
    nnz: int
    density: float
    mode_order: tuple
    slice_count: int
    fiber_count: int
    mean_nnz_per_slice: float
    stddev_nnz_per_slice: float
    max_nnz_per_slice: int
    mean_nnz_per_fiber: float
    stddev_nnz_per_fiber: float
    max_nnz_per_fiber: int

    def to_dict(self) -> dict:
        d = dict(self.__dict__)
        d["dims"] = list(self.dims)
        d["mode_order"] = list(self.mode_order)
        return d


def compute_stats(t: CooTensor, mode_order: Sequence[int] | None = None) -> TensorStats:
    """Statistics under ``mode_order`` (identity by default), coo.py:281-325.
    Duplicate coordinates count as distinct entries, as in the reference."""
    mo = _check_mode_order(mode_order, t.order) if mode_order is not None else tuple(range(t.order))
    density = t.nnz / math.prod(float(d) for d in t.dims)
    if t.nnz == 0:
        return TensorStats(order=t.order, dims=t.dims, nnz=0, density=0.0, mode_order=mo,
                           slice_count=0, fiber_count=0, mean_nnz_per_slice=0.0,
                           stddev_nnz_per_slice=0.0, max_nnz_per_slice=0, mean_nnz_per_fiber=0.0,
                           stddev_nnz_per_fiber=0.0, max_nnz_per_fiber=0)
    pop = population(build_csf(t, mo))
    ms, ss = mean_std(pop.nnz, pop.sumsq_slice, pop.slices)
    mf, sf = mean_std(pop.nnz, pop.sumsq_fiber, pop.fibers)
    return TensorStats(
        order=t.order, dims=t.dims, nnz=t.nnz, density=density, mode_order=mo,
        slice_count=int(pop.slices), fiber_count=int(pop.fibers),
        mean_nnz_per_slice=ms, stddev_nnz_per_slice=ss, max_nnz_per_slice=int(pop.max_slice),
        mean_nnz_per_fiber=mf, stddev_nnz_per_fiber=sf, max_nnz_per_fiber=int(pop.max_fiber),
    )
