"""CSF, CSL and HB-CSF containers backed by device arrays.

Mirrors ``tenkit.formats`` (pkg/src/tenkit/formats.py).  ``build_csf`` and
``build_hbcsf`` run the on-GPU builder in libhbk (K1-K3); the containers hold
native handles and expose the reference's attributes (``ptrs``, ``idxs``,
``leaf_idx``, ``values``, ``slice_ptr`` …) as host arrays fetched on first
access, in the reference's dtypes (int64 pointers, uint32 indices, float64
values).  Those arrays are bit-identical to the reference builder's output.
"""
from __future__ import annotations

import ctypes as C
import enum
import math
from dataclasses import dataclass
from functools import singledispatch
from typing import Sequence

import numpy as np

from . import _native as N
from .coo import INDEX_DTYPE, VALUE_DTYPE, CooTensor, _check_mode_order

PTR_DTYPE = np.int64
INDEX_WORD_BYTES = 4


class SliceKind(enum.IntEnum):
    """Bucket a slice lands in (formats.py:41-46)."""

    COO = 0
    CSL = 1
    CSF = 2


class CsfTensor:
    """Compressed sparse fiber tree (formats.py:49-117), device-resident."""

    __slots__ = ("_h", "_info", "_cache", "_plans", "__weakref__")

    def __init__(self, handle: N.Handle):
        self._h = handle
        info = N.CsfInfo()
        N.call("hbk_csf_info_get", handle.ptr, C.byref(info))
        self._info = info
        self._cache = {}
        self._plans = {}

    @property
    def dims(self) -> tuple[int, ...]:
        return tuple(int(self._info.dims[d]) for d in range(self._info.order))

    @property
    def mode_order(self) -> tuple[int, ...]:
        return tuple(int(self._info.mode_order[d]) for d in range(self._info.order))

    @property
    def split(self) -> bool:
        return bool(self._info.split)

    @property
    def order(self) -> int:
        return int(self._info.order)

    @property
    def nnz(self) -> int:
        return int(self._info.nnz)

    def level_sizes(self) -> tuple[int, ...]:
        return tuple(int(self._info.level_sizes[d]) for d in range(self.order - 1))

    @property
    def num_slices(self) -> int:
        return self.level_sizes()[0]

    @property
    def num_fibers(self) -> int:
        """Leaf-parent nodes (level N-2); segments count separately after a split."""
        return self.level_sizes()[-1]

    def _export(self, which: int, level: int, dtype, count: int) -> np.ndarray:
        key = (which, level)
        arr = self._cache.get(key)
        if arr is None:
            arr = np.empty(count, dtype=dtype)
            N.call("hbk_csf_export", self._h.ptr, which, level,
                   arr.ctypes.data_as(C.c_void_p), N.stream_ptr())
            self._cache[key] = arr
        return arr

    @property
    def ptrs(self) -> tuple[np.ndarray, ...]:
        ls = self.level_sizes()
        return tuple(self._export(N.HBK_CSF_PTR, d, PTR_DTYPE, ls[d] + 1) for d in range(self.order - 1))

    @property
    def idxs(self) -> tuple[np.ndarray, ...]:
        ls = self.level_sizes()
        return tuple(self._export(N.HBK_CSF_IDX, d, INDEX_DTYPE, ls[d]) for d in range(self.order - 1))

    @property
    def leaf_idx(self) -> np.ndarray:
        return self._export(N.HBK_CSF_LEAF, 0, INDEX_DTYPE, self.nnz)

    @property
    def values(self) -> np.ndarray:
        return self._export(N.HBK_CSF_VALUES, 0, VALUE_DTYPE, self.nnz)

    # host-side structural views (formats.py:102-117), over the exported arrays
    def fiber_positions(self) -> np.ndarray:
        pos = self.ptrs[0]
        for d in range(1, self.order - 2):
            pos = self.ptrs[d][pos]
        return pos

    def leaf_offsets(self) -> np.ndarray:
        return self.ptrs[-1][self.fiber_positions()]

    def slice_nnz(self) -> np.ndarray:
        return np.diff(self.leaf_offsets())

    def fiber_sizes(self) -> np.ndarray:
        return np.diff(self.ptrs[-1])

    def __repr__(self) -> str:
        return (f"CsfTensor(dims={self.dims}, mode_order={self.mode_order}, nnz={self.nnz}, "
                f"levels={self.level_sizes()}, split={self.split})")


class CslSlices:
    """Slices whose fiber level is skipped (formats.py:207-233), device-resident."""

    __slots__ = ("_h", "_info", "_cache", "_plans", "__weakref__")

    def __init__(self, handle: N.Handle):
        self._h = handle
        info = N.CslInfo()
        N.call("hbk_csl_info_get", handle.ptr, C.byref(info))
        self._info = info
        self._cache = {}
        self._plans = {}

    @property
    def dims(self) -> tuple[int, ...]:
        return tuple(int(self._info.dims[d]) for d in range(self._info.order))

    @property
    def mode_order(self) -> tuple[int, ...]:
        return tuple(int(self._info.mode_order[d]) for d in range(self._info.order))

    @property
    def order(self) -> int:
        return int(self._info.order)

    @property
    def nnz(self) -> int:
        return int(self._info.nnz)

    @property
    def num_slices(self) -> int:
        return int(self._info.num_slices)

    def _export(self, which: int, dtype, shape) -> np.ndarray:
        arr = self._cache.get(which)
        if arr is None:
            arr = np.empty(shape, dtype=dtype)
            N.call("hbk_csl_export", self._h.ptr, which, arr.ctypes.data_as(C.c_void_p),
                   N.stream_ptr())
            self._cache[which] = arr
        return arr

    @property
    def slice_ptr(self) -> np.ndarray:
        return self._export(N.HBK_CSL_SLICE_PTR, PTR_DTYPE, self.num_slices + 1)

    @property
    def slice_idx(self) -> np.ndarray:
        return self._export(N.HBK_CSL_SLICE_IDX, INDEX_DTYPE, self.num_slices)

    @property
    def rest_idx(self) -> np.ndarray:
        return self._export(N.HBK_CSL_REST_IDX, INDEX_DTYPE, (self.nnz, self.order - 1))

    @property
    def values(self) -> np.ndarray:
        return self._export(N.HBK_CSL_VALUES, VALUE_DTYPE, self.nnz)

    def __repr__(self) -> str:
        return f"CslSlices(dims={self.dims}, mode_order={self.mode_order}, slices={self.num_slices}, nnz={self.nnz})"


class HbCsfTensor:
    """Hybrid format: per-slice routing into COO, CSL and CSF buckets
    (formats.py:236-257).  The buckets are slice-disjoint."""

    __slots__ = ("dims", "mode_order", "coo_part", "csl_part", "csf_part", "_plans", "__weakref__")

    def __init__(self, dims, mode_order, coo_part: CooTensor, csl_part: CslSlices, csf_part: CsfTensor):
        self.dims = tuple(dims)
        self.mode_order = tuple(mode_order)
        self.coo_part = coo_part
        self.csl_part = csl_part
        self.csf_part = csf_part
        self._plans = {}

    @property
    def order(self) -> int:
        return len(self.dims)

    @property
    def nnz(self) -> int:
        return self.coo_part.nnz + self.csl_part.nnz + self.csf_part.nnz

    def census(self) -> dict[str, int]:
        return slice_census(self)

    def __repr__(self) -> str:
        return (f"HbCsfTensor(dims={self.dims}, mode_order={self.mode_order}, "
                f"coo={self.coo_part.nnz}, csl={self.csl_part.nnz}, csf={self.csf_part.nnz})")


def build_csf(t: CooTensor, mode_order: Sequence[int]) -> CsfTensor:
    """Compress a canonical COO tensor into a CSF tree on the GPU (formats.py:120-168)."""
    mo = _check_mode_order(mode_order, t.order)
    out = N.new_out()
    N.call("hbk_build_csf", t._dev().ptr, N.int_array(mo), N.stream_ptr(), C.byref(out))
    return CsfTensor(N.Handle(out, "hbk_csf_release"))


def build_hbcsf(t: CooTensor, mode_order: Sequence[int]) -> HbCsfTensor:
    """Route each slice into the hybrid's three buckets on the GPU (formats.py:260-299)."""
    mo = _check_mode_order(mode_order, t.order)
    coo, csl, csf = N.new_out(), N.new_out(), N.new_out()
    N.call("hbk_build_hbcsf", t._dev().ptr, N.int_array(mo), N.stream_ptr(), C.byref(coo),
           C.byref(csl), C.byref(csf))
    return HbCsfTensor(
        t.dims, mo,
        CooTensor._from_handle(N.Handle(coo, "hbk_coo_release")),
        CslSlices(N.Handle(csl, "hbk_csl_release")),
        CsfTensor(N.Handle(csf, "hbk_csf_release")),
    )


def classify_slices(c: CsfTensor) -> np.ndarray:
    """int8 SliceKind label per slice (formats.py:194-204), computed on the GPU."""
    labels = np.empty(c.num_slices, dtype=np.int8)
    if c.num_slices:
        N.call("hbk_classify_slices", c._h.ptr, labels.ctypes.data_as(C.c_void_p), N.stream_ptr())
    return labels


def population(c: CsfTensor) -> N.Population:
    """Slice/fiber population counts of a tree, reduced on the GPU
    (hbk_csf_population): sizes, maxima, exact sums of squares, classes."""
    pop = N.Population()
    N.call("hbk_csf_population", c._h.ptr, C.byref(pop), N.stream_ptr())
    return pop


def mean_std(total: int, sumsq: int, count: int) -> tuple[float, float]:
    """Mean and population standard deviation from exact integer moments."""
    if count == 0:
        return 0.0, 0.0
    var_num = count * int(sumsq) - int(total) * int(total)  # exact: count^2 * variance
    return total / count, math.sqrt(max(var_num, 0) / (count * count))


def slice_census(x) -> dict[str, int]:
    """Slices per bucket (formats.py:315-328); a tree's classes are counted
    on the GPU."""
    if isinstance(x, CsfTensor):
        pop = population(x)
        return {"coo": int(pop.coo_slices), "csl": int(pop.csl_slices), "csf": int(pop.csf_slices)}
    return {"coo": x.coo_part.nnz, "csl": x.csl_part.num_slices, "csf": x.csf_part.num_slices}


@dataclass(frozen=True)
class StoragePart:
    label: str
    slices: int
    fibers: int
    nnz: int
    words: int

    def to_dict(self) -> dict:
        return dict(self.__dict__)


@dataclass(frozen=True)
class StorageReport:
    """32-bit index-word accounting (formats.py:343-365)."""

    format: str
    index_words: int
    parts: tuple[StoragePart, ...]

    @property
    def index_bytes(self) -> int:
        return self.index_words * INDEX_WORD_BYTES

    def to_dict(self) -> dict:
        return {"format": self.format, "index_words": self.index_words,
                "index_bytes": self.index_bytes, "parts": [p.to_dict() for p in self.parts]}


@singledispatch
def storage_words(x) -> StorageReport:
    """Index words of a representation (formats.py:368-415), from its sizes."""
    raise TypeError(f"no storage accounting for {type(x).__name__}")


@storage_words.register
def _(x: CooTensor) -> StorageReport:
    words = x.order * x.nnz
    if x.nnz == 0:
        s = f = 0
    else:
        # distinct leading coordinates / leading (order-1)-tuples under the
        # tensor's order = the level sizes of its CSF tree, built on the GPU
        mo = x.sorted_under if x.sorted_under is not None else tuple(range(x.order))
        ls = build_csf(x, mo).level_sizes()
        s, f = ls[0], ls[-1]
    return StorageReport("coo", words, (StoragePart("coo", s, f, x.nnz, words),))


@storage_words.register
def _(x: CsfTensor) -> StorageReport:
    words = sum(2 * n for n in x.level_sizes()) + x.nnz
    return StorageReport("csf", words, (StoragePart("csf", x.num_slices, x.num_fibers, x.nnz, words),))


@storage_words.register
def _(x: CslSlices) -> StorageReport:
    words = 2 * x.num_slices + (x.order - 1) * x.nnz
    return StorageReport("csl", words, (StoragePart("csl", x.num_slices, x.nnz, x.nnz, words),))


@storage_words.register
def _(x: HbCsfTensor) -> StorageReport:
    coo_words = x.order * x.coo_part.nnz
    coo = StoragePart("coo", x.coo_part.nnz, x.coo_part.nnz, x.coo_part.nnz, coo_words)
    csl = storage_words(x.csl_part).parts[0]
    csf = storage_words(x.csf_part).parts[0]
    return StorageReport("hbcsf", coo.words + csl.words + csf.words, (coo, csl, csf))
