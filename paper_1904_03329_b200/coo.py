"""Coordinate (COO) tensors — the input side of the HB-CSF path.

Mirrors the reference container ``tenkit.coo`` (pkg/src/tenkit/coo.py):
same constructor, validation, attribute names and exceptions.  The arrays
live on the host as in the reference *and* (lazily) on the GPU as an
``hbk_coo`` handle; every transformation (sort, canonicalize) runs on the
GPU through libhbk and returns a tensor whose host arrays are fetched only if
someone reads them.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Iterator, Sequence

import numpy as np

from . import _native as N

INDEX_DTYPE = np.uint32
VALUE_DTYPE = np.float64


class ParseError(ValueError):
    """Malformed tensor text (coo.py:21-28).  Carries the 1-based line number."""

    def __init__(self, message: str, line: int | None = None):
        if line is not None:
            message = f"line {line}: {message}"
        super().__init__(message)
        self.line = line


class CapacityError(ValueError):
    """A requested dense intermediate would exceed the configured ceiling (coo.py:31-32)."""


def _check_mode_order(mode_order: Sequence[int], order: int) -> tuple[int, ...]:
    """coo.py:35-39."""
    mo = tuple(int(m) for m in mode_order)
    if sorted(mo) != list(range(order)):
        raise ValueError(f"mode_order {mo} is not a permutation of 0..{order - 1}")
    return mo


def _is_cuda_tensor(x) -> bool:
    mod = type(x).__module__
    return mod.startswith("torch") and getattr(x, "is_cuda", False)


class CooTensor:
    """Sparse tensor in coordinate form (coo.py:42-114).

    ``indices`` is (nnz, order) uint32, ``values`` (nnz,) float64,
    ``sorted_under`` the mode order the entries are sorted under (or None).
    ``indices``/``values`` may also be CUDA tensors (uint32/int32/int64 and
    float32/float64), in which case the tensor is created on the device and
    host copies are made only on demand.  Treat instances as immutable.
    """

    __slots__ = ("_dims", "_indices", "_values", "_sorted_under", "_handle", "_nnz",
                 "_slice_views", "_plans", "__weakref__")

    def __init__(self, dims, indices, values, sorted_under=None):
        dims = tuple(int(d) for d in dims)
        if len(dims) < 3:
            raise ValueError(f"tensor order must be >= 3, got {len(dims)}")
        if any(d < 1 for d in dims):
            raise ValueError(f"all dimensions must be positive, got {dims}")
        self._handle = None
        self._slice_views = {}
        self._plans = {}
        so = None if sorted_under is None else _check_mode_order(sorted_under, len(dims))
        self._dims = dims
        self._sorted_under = so
        if _is_cuda_tensor(indices):
            self._init_device(indices, values)
            return
        idx = np.asarray(indices)
        if idx.ndim != 2 or idx.shape[1] != len(dims):
            raise ValueError(f"indices must have shape (nnz, {len(dims)}), got {idx.shape}")
        vals = np.asarray(values, dtype=VALUE_DTYPE)
        if vals.shape != (idx.shape[0],):
            raise ValueError("values length does not match indices")
        if idx.size:
            lo = idx.min(axis=0)
            hi = idx.max(axis=0)
            if lo.min() < 0 or any(int(h) >= d for h, d in zip(hi, dims)):
                raise ValueError("index out of range for dims")
        self._indices = np.ascontiguousarray(idx, dtype=INDEX_DTYPE)
        self._values = vals
        self._nnz = int(vals.shape[0])

    def _init_device(self, indices, values):
        torch = N.require_device()
        dims = self._dims
        if indices.dim() != 2 or indices.shape[1] != len(dims):
            raise ValueError(f"indices must have shape (nnz, {len(dims)}), got {tuple(indices.shape)}")
        if values.dim() != 1 or values.shape[0] != indices.shape[0]:
            raise ValueError("values length does not match indices")
        nnz = int(indices.shape[0])
        if nnz:
            lo = indices.amin(dim=0).cpu()
            hi = indices.amax(dim=0).cpu()
            if int(lo.min()) < 0 or any(int(h) >= d for h, d in zip(hi.tolist(), dims)):
                raise ValueError("index out of range for dims")
        idx = indices.to(torch.int32).contiguous() if indices.dtype != torch.int32 else indices.contiguous()
        so = N.int_array(self._sorted_under) if self._sorted_under is not None else None
        out = N.new_out()
        if values.dtype == torch.float64:
            v = values.contiguous()
            N.call("hbk_coo_create", len(dims), N.i64_array(dims), nnz, C.c_void_p(idx.data_ptr()),
                   C.c_void_p(v.data_ptr()), so, N.stream_ptr(), C.byref(out))
        else:
            v = values.to(torch.float32).contiguous()
            N.call("hbk_coo_create_f32", len(dims), N.i64_array(dims), nnz,
                   C.c_void_p(idx.data_ptr()), C.c_void_p(v.data_ptr()), so, N.stream_ptr(),
                   C.byref(out))
        self._handle = N.Handle(out, "hbk_coo_release")
        self._indices = None
        self._values = None
        self._nnz = nnz

    @classmethod
    def _from_handle(cls, handle: N.Handle) -> "CooTensor":
        info = N.CooInfo()
        N.call("hbk_coo_info_get", handle.ptr, C.byref(info))
        self = object.__new__(cls)
        self._dims = tuple(int(info.dims[d]) for d in range(info.order))
        self._sorted_under = (
            tuple(int(info.sorted_under[d]) for d in range(info.order)) if info.has_sorted else None
        )
        self._handle = handle
        self._indices = None
        self._values = None
        self._nnz = int(info.nnz)
        self._slice_views = {}
        self._plans = {}
        return self

    # ---------------------------------------------------------- attributes
    @property
    def dims(self) -> tuple[int, ...]:
        return self._dims

    @property
    def sorted_under(self) -> tuple[int, ...] | None:
        return self._sorted_under

    @property
    def indices(self) -> np.ndarray:
        if self._indices is None:
            self._fetch()
        return self._indices

    @property
    def values(self) -> np.ndarray:
        if self._values is None:
            self._fetch()
        return self._values

    def _fetch(self) -> None:
        idx = np.empty((self._nnz, len(self._dims)), dtype=INDEX_DTYPE)
        vals = np.empty(self._nnz, dtype=VALUE_DTYPE)
        if self._nnz:
            N.call("hbk_coo_export", self._handle.ptr, idx.ctypes.data_as(C.c_void_p),
                   vals.ctypes.data_as(C.c_void_p), N.stream_ptr())
        self._indices, self._values = idx, vals

    @property
    def order(self) -> int:
        return len(self._dims)

    @property
    def nnz(self) -> int:
        return self._nnz

    def entries(self) -> Iterator[tuple[tuple[int, ...], float]]:
        for row, v in zip(self.indices, self.values):
            yield tuple(int(i) for i in row), float(v)

    def __eq__(self, other) -> bool:
        if not isinstance(other, CooTensor):
            return NotImplemented
        return (
            self.dims == other.dims
            and np.array_equal(self.indices, other.indices)
            and np.array_equal(self.values, other.values)
        )

    __hash__ = None

    def __repr__(self) -> str:
        return f"CooTensor(dims={self.dims}, nnz={self.nnz}, sorted_under={self.sorted_under})"

    # ------------------------------------------------------------- device
    def _dev(self) -> N.Handle:
        """The device-resident copy (uploaded on first use)."""
        if self._handle is None:
            torch = N.require_device()
            idx = torch.from_numpy(self._indices.view(np.int32)).cuda()
            vals = torch.from_numpy(self._values).cuda()
            so = N.int_array(self._sorted_under) if self._sorted_under is not None else None
            out = N.new_out()
            N.call("hbk_coo_create", self.order, N.i64_array(self._dims), self._nnz,
                   C.c_void_p(idx.data_ptr()), C.c_void_p(vals.data_ptr()), so, N.stream_ptr(),
                   C.byref(out))
            self._handle = N.Handle(out, "hbk_coo_release")
        return self._handle

    def _slices(self, mode: int):
        """CSL-shaped slice view of this tensor for mode (mttkrp_coo path)."""
        h = self._slice_views.get(mode)
        if h is None:
            out = N.new_out()
            N.call("hbk_coo_slices", self._dev().ptr, int(mode), N.stream_ptr(), C.byref(out))
            h = N.Handle(out, "hbk_csl_release")
            self._slice_views[mode] = h
        return h


def sort_by_mode_order(t: CooTensor, mode_order: Sequence[int]) -> CooTensor:
    """Stable lexicographic sort, mode_order[0] major (coo.py:214-224), on the GPU."""
    mo = _check_mode_order(mode_order, t.order)
    if t.sorted_under == mo:
        return t
    out = N.new_out()
    N.call("hbk_coo_sort", t._dev().ptr, N.int_array(mo), N.stream_ptr(), C.byref(out))
    return CooTensor._from_handle(N.Handle(out, "hbk_coo_release"))


def canonicalize(t: CooTensor) -> CooTensor:
    """Identity sort, duplicates summed, exact zeros dropped (coo.py:227-247), on the GPU.

    Duplicate runs are summed in np.add.reduceat's association order, so the
    result is bit-identical to the reference's."""
    identity = tuple(range(t.order))
    if t.nnz == 0:
        return CooTensor(t.dims, t.indices, t.values, sorted_under=identity)
    out = N.new_out()
    N.call("hbk_coo_canonicalize", t._dev().ptr, 0, N.stream_ptr(), C.byref(out))
    return CooTensor._from_handle(N.Handle(out, "hbk_coo_release"))


def unique_coordinates(t: CooTensor) -> CooTensor:
    """Identity-sorted, duplicates dropped keeping the first (set semantics)."""
    out = N.new_out()
    N.call("hbk_coo_canonicalize", t._dev().ptr, 1, N.stream_ptr(), C.byref(out))
    return CooTensor._from_handle(N.Handle(out, "hbk_coo_release"))


def allmode_order(dims: Sequence[int], mode: int) -> tuple[int, ...]:
    """Target mode first, then the other modes by ascending dimension, ties by
    mode id (coo.py:328-336)."""
    n = len(dims)
    if not 0 <= mode < n:
        raise ValueError(f"mode {mode} out of range for order {n}")
    rest = sorted((d for d in range(n) if d != mode), key=lambda d: (dims[d], d))
    return (mode, *rest)


# ---------------------------------------------------------------- FROSTT text
def _tns_to_tensor(handle) -> "CooTensor":
    order = C.c_int()
    nnz = C.c_int64()
    dims = (C.c_int64 * N.HBK_MAX_ORDER)()
    N.call("hbk_tns_info", handle, C.byref(order), C.byref(nnz), dims, None)
    o, m = int(order.value), int(nnz.value)
    idx = np.empty((m, o), dtype=INDEX_DTYPE)
    vals = np.empty(m, dtype=VALUE_DTYPE)
    N.call("hbk_tns_export", handle, idx.ctypes.data_as(C.c_void_p), vals.ctypes.data_as(C.c_void_p))
    return CooTensor(tuple(int(dims[d]) for d in range(o)), idx, vals)


def _tns_call(fn, *args) -> "CooTensor":
    lib = N.lib()
    h = C.c_void_p()
    status = getattr(lib, fn)(*args, C.byref(h))
    try:
        if status != N.HBK_OK:
            msg = lib.hbk_last_error().decode(errors="replace")
            line = C.c_int64(0)
            if h:
                lib.hbk_tns_info(h, None, None, None, C.byref(line))
            if status == N.HBK_EINVAL:
                raise ParseError(msg, int(line.value) if line.value else None)
            N.check(status)
        return _tns_to_tensor(h)
    finally:
        if h:
            lib.hbk_tns_release(h)


def _dims_arg(dims):
    if dims is None:
        return 0, None
    d = tuple(int(x) for x in dims)
    if len(d) < 3:
        raise ValueError(f"tensor order must be >= 3, got {len(d)}")
    return len(d), N.i64_array(d)


def parse_frostt(stream, dims: Sequence[int] | None = None, *, threads: int = 0) -> CooTensor:
    """Parse FROSTT text into a CooTensor (coo.py:117-184), in libhbk's
    multi-threaded host parser: '#' comments, blank lines skipped, 1-based
    indices, order from the first data line unless ``dims`` is given.
    Raises ParseError with the 1-based line of the first malformed line."""
    order, darr = _dims_arg(dims)
    text = stream if isinstance(stream, (str, bytes, bytearray)) else stream.read()
    data = text.encode("utf-8") if isinstance(text, str) else bytes(text)
    return _tns_call("hbk_tns_parse", data, len(data), order, darr, int(threads))


def load_frostt(path: str, dims: Sequence[int] | None = None, *, threads: int = 0) -> CooTensor:
    """Read and parse a .tns file (coo.py:198-200); the file is read and parsed in C++."""
    order, darr = _dims_arg(dims)
    return _tns_call("hbk_tns_load", os.fsencode(path), order, darr, int(threads))


def _tns_text(t: CooTensor, threads: int = 0) -> bytes:
    idx = np.ascontiguousarray(t.indices, dtype=INDEX_DTYPE)
    vals = np.ascontiguousarray(t.values, dtype=VALUE_DTYPE)
    ptr = C.c_void_p()
    n = C.c_int64()
    N.call("hbk_tns_format", idx.ctypes.data_as(C.c_void_p), vals.ctypes.data_as(C.c_void_p),
           int(t.nnz), int(t.order), int(threads), C.byref(ptr), C.byref(n))
    try:
        return C.string_at(ptr, n.value)
    finally:
        N.lib().hbk_tns_free_text(ptr)


def write_frostt(t: CooTensor, stream) -> None:
    """FROSTT text (coo.py:187-195): 1-based indices, values with 17
    significant digits (round-trip exact), entries in the tensor's order."""
    text = _tns_text(t)
    try:
        stream.write(text.decode("ascii"))
    except TypeError:
        stream.write(text)


def save_frostt(t: CooTensor, path: str) -> None:
    """Write a .tns file (coo.py:203-205)."""
    with open(path, "wb") as fh:
        fh.write(_tns_text(t))
