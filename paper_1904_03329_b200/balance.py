"""B-CSF load balancing: fiber splitting and slice-to-block schedules.

Mirrors ``tenkit.balance`` (pkg/src/tenkit/balance.py).  ``split_fibers``
(K4) and ``assign_slice_blocks`` (K5) run on the GPU and produce the same
arrays/units as the reference; a schedule can be handed to
``mttkrp_scheduled``/``mttkrp_hbcsf``, whose CSF work units are then exactly
its units.
"""
from __future__ import annotations

import ctypes as C
import weakref
from dataclasses import dataclass
from functools import singledispatch

import numpy as np

from . import _native as N
from .formats import CsfTensor, HbCsfTensor


@dataclass(frozen=True)
class SplitConfig:
    """Fiber threshold and block nonzero budget (balance.py:27-48)."""

    fiber_threshold: int = 128
    block_size: int = 512
    warp_size: int = 32

    def __post_init__(self):
        if self.fiber_threshold < 1:
            raise ValueError("fiber_threshold must be at least 1")
        if self.warp_size < 1:
            raise ValueError("warp_size must be at least 1")
        if self.block_size < 1 or self.block_size % self.warp_size != 0:
            raise ValueError(
                f"block_size {self.block_size} must be a positive multiple of "
                f"warp_size {self.warp_size}"
            )


@singledispatch
def split_fibers(t, cfg: SplitConfig):
    """Cut fibers longer than cfg.fiber_threshold into segments (balance.py:51-97).

    Returns the input object itself when no fiber exceeds the threshold."""
    raise TypeError(f"cannot split {type(t).__name__}")


@split_fibers.register
def _(t: CsfTensor, cfg: SplitConfig) -> CsfTensor:
    out = N.new_out()
    N.call("hbk_split_fibers", t._h.ptr, int(cfg.fiber_threshold), N.stream_ptr(), C.byref(out))
    if not out.value:
        return t
    return CsfTensor(N.Handle(out, "hbk_csf_release"))


@split_fibers.register
def _(t: HbCsfTensor, cfg: SplitConfig) -> HbCsfTensor:
    # only the CSF bucket has multi-nonzero fibers (balance.py:93-97)
    return HbCsfTensor(t.dims, t.mode_order, t.coo_part, t.csl_part, split_fibers(t.csf_part, cfg))


@dataclass(frozen=True)
class ScheduleUnit:
    """One thread block's work: a contiguous run of fibers of one slice."""

    block_id: int
    slice_pos: int
    fiber_start: int
    fiber_stop: int


class BlockSchedule:
    """Slice-major assignment of fiber runs to blocks (balance.py:110-150).

    Built by ``assign_slice_blocks`` (device handle, units fetched lazily) or
    directly from host ``units``/``multiplicities`` like the reference."""

    def __init__(self, units=None, multiplicities=None, num_slices: int = 0, num_fibers: int = 0,
                 *, _handle: N.Handle | None = None):
        self._handle = _handle
        self._bound = weakref.WeakKeyDictionary()  # tree -> device schedule
        if _handle is not None:
            info = N.SchedInfo()
            N.call("hbk_sched_info_get", _handle.ptr, C.byref(info))
            self.num_slices = int(info.num_slices)
            self.num_fibers = int(info.num_fibers)
            self._num_units = int(info.num_units)
            self._units = None
            self._mult = None
        else:
            self._units = tuple(units)
            self._mult = np.asarray(multiplicities, dtype=np.int64)
            self.num_slices = int(num_slices)
            self.num_fibers = int(num_fibers)
            self._num_units = len(self._units)

    @property
    def units(self) -> tuple[ScheduleUnit, ...]:
        if self._units is None:
            raw = np.empty((self._num_units, 4), dtype=np.int64)
            if self._num_units:
                N.call("hbk_sched_export", self._handle.ptr, N.HBK_SCHED_UNITS,
                       raw.ctypes.data_as(C.c_void_p), N.stream_ptr())
            self._units = tuple(ScheduleUnit(*map(int, r)) for r in raw)
        return self._units

    @property
    def multiplicities(self) -> np.ndarray:
        if self._mult is None:
            m = np.empty(self.num_slices, dtype=np.int64)
            if self.num_slices:
                N.call("hbk_sched_export", self._handle.ptr, N.HBK_SCHED_MULT,
                       m.ctypes.data_as(C.c_void_p), N.stream_ptr())
            self._mult = m
        return self._mult

    @property
    def num_blocks(self) -> int:
        return self._num_units

    def units_array(self) -> np.ndarray:
        """Units as an int64 (num_units, 4) array (block_id, slice_pos, start, stop)."""
        if self._handle is not None:
            raw = np.empty((self._num_units, 4), dtype=np.int64)
            if self._num_units:
                N.call("hbk_sched_export", self._handle.ptr, N.HBK_SCHED_UNITS,
                       raw.ctypes.data_as(C.c_void_p), N.stream_ptr())
            return raw
        return np.array([[u.block_id, u.slice_pos, u.fiber_start, u.fiber_stop] for u in self._units],
                        dtype=np.int64).reshape(-1, 4)

    def _device_for(self, t: CsfTensor) -> N.Handle:
        """Device schedule usable with tree t (uploaded for host-built schedules)."""
        if self._handle is not None:
            return self._handle
        h = self._bound.get(t)
        if h is None:
            raw = np.ascontiguousarray(self.units_array())
            mult = np.ascontiguousarray(self._mult, dtype=np.int64)
            out = N.new_out()
            N.call("hbk_sched_from_units", t._h.ptr, raw.ctypes.data_as(C.c_void_p), len(raw),
                   mult.ctypes.data_as(C.c_void_p) if mult.size else None, N.stream_ptr(),
                   C.byref(out))
            h = N.Handle(out, "hbk_sched_release")
            self._bound[t] = h
        return h

    def validate_for(self, t: CsfTensor) -> None:
        """Raise ValueError unless this schedule partitions t's fibers (balance.py:128-150)."""
        if t.num_slices != self.num_slices or t.num_fibers != self.num_fibers:
            raise ValueError(
                f"schedule was built for {self.num_slices} slices/"
                f"{self.num_fibers} fibers, tensor has {t.num_slices}/{t.num_fibers}"
            )
        N.call("hbk_sched_validate", self._device_for(t).ptr, t._h.ptr, N.stream_ptr())


def assign_slice_blocks(t: CsfTensor, cfg: SplitConfig) -> BlockSchedule:
    """Multiplicity max(1, ceil(m/block_size)) per slice and greedy fiber-run
    units (balance.py:153-189), computed on the GPU."""
    out = N.new_out()
    N.call("hbk_assign_slice_blocks", t._h.ptr, int(cfg.block_size), N.stream_ptr(), C.byref(out))
    return BlockSchedule(_handle=N.Handle(out, "hbk_sched_release"))


@dataclass(frozen=True)
class ImbalanceMetrics:
    """Population spread of nonzeros over slices and fibers (balance.py:192-207)."""

    slices: int
    fibers: int
    nnz: int
    mean_nnz_per_slice: float
    stddev_nnz_per_slice: float
    max_nnz_per_slice: int
    mean_nnz_per_fiber: float
    stddev_nnz_per_fiber: float
    max_nnz_per_fiber: int

    def to_dict(self) -> dict:
        return dict(self.__dict__)


def imbalance_metrics(t: CsfTensor) -> ImbalanceMetrics:
    """Mean, population stddev and max of nonzeros per slice and per fiber
    (per segment once split), balance.py:210-227.  Reduced on the GPU over
    the tree's pointer arrays (hbk_csf_population, exact integer moments)."""
    from .formats import mean_std, population

    if t.nnz == 0:
        return ImbalanceMetrics(0, 0, 0, 0.0, 0.0, 0, 0.0, 0.0, 0)
    pop = population(t)
    ms, ss = mean_std(pop.nnz, pop.sumsq_slice, pop.slices)
    mf, sf = mean_std(pop.nnz, pop.sumsq_fiber, pop.fibers)
    return ImbalanceMetrics(
        slices=int(pop.slices), fibers=int(pop.fibers), nnz=int(pop.nnz),
        mean_nnz_per_slice=ms, stddev_nnz_per_slice=ss, max_nnz_per_slice=int(pop.max_slice),
        mean_nnz_per_fiber=mf, stddev_nnz_per_fiber=sf, max_nnz_per_fiber=int(pop.max_fiber),
    )
