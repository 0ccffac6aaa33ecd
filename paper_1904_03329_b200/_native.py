"""ctypes binding of libhbk.so (include/hbk.h).

The shared library is built in-tree by ``__graft_entry__.build()`` (or
``python -m paper_1904_03329_b200.build``).  There is no CPU fallback: if the
library or a CUDA device is missing, every entry point raises.
"""
from __future__ import annotations

import ctypes as C
import os
import threading
from pathlib import Path

_HERE = Path(__file__).resolve().parent
LIB_PATH = _HERE / "libhbk.so"

HBK_MAX_ORDER = 8
HBK_OK, HBK_EINVAL, HBK_ETYPE, HBK_ECUDA, HBK_ENOMEM = 0, 1, 2, 3, 4

HBK_CSL_SLICE_PTR, HBK_CSL_SLICE_IDX, HBK_CSL_REST_IDX, HBK_CSL_VALUES = 0, 1, 2, 3
HBK_CSF_PTR, HBK_CSF_IDX, HBK_CSF_LEAF, HBK_CSF_VALUES = 0, 1, 2, 3
HBK_SCHED_UNITS, HBK_SCHED_MULT = 0, 1

i64 = C.c_int64
vp = C.c_void_p


class CooInfo(C.Structure):
    _fields_ = [
        ("order", C.c_int),
        ("dims", i64 * HBK_MAX_ORDER),
        ("nnz", i64),
        ("has_sorted", C.c_int),
        ("sorted_under", C.c_int * HBK_MAX_ORDER),
        ("unique_mode", C.c_int),
    ]


class CslInfo(C.Structure):
    _fields_ = [
        ("order", C.c_int),
        ("dims", i64 * HBK_MAX_ORDER),
        ("mode_order", C.c_int * HBK_MAX_ORDER),
        ("num_slices", i64),
        ("nnz", i64),
    ]


class CsfInfo(C.Structure):
    _fields_ = [
        ("order", C.c_int),
        ("dims", i64 * HBK_MAX_ORDER),
        ("mode_order", C.c_int * HBK_MAX_ORDER),
        ("nnz", i64),
        ("level_sizes", i64 * HBK_MAX_ORDER),
        ("split", C.c_int),
    ]


class Population(C.Structure):
    _fields_ = [
        ("slices", i64), ("fibers", i64), ("nnz", i64),
        ("max_slice", i64), ("max_fiber", i64),
        ("sumsq_slice", C.c_uint64), ("sumsq_fiber", C.c_uint64),
        ("coo_slices", i64), ("csl_slices", i64), ("csf_slices", i64),
    ]


class SchedInfo(C.Structure):
    _fields_ = [
        ("num_units", i64),
        ("num_slices", i64),
        ("num_fibers", i64),
        ("block_size", i64),
    ]


class PlanInfo(C.Structure):
    _fields_ = [
        ("mode", C.c_int),
        ("rank", C.c_int),
        ("out_rows", i64),
        ("tasks_csf", i64),
        ("tasks_csl", i64),
        ("tasks_coo", i64),
        ("tasks_zero", i64),
        ("split_rows", i64),
        ("launches", i64),
        ("fast_path", C.c_int),
        ("op_muls", i64),
        ("op_adds", i64),
        ("nnz", i64),
        ("stream_bytes", i64),
        ("tasks_heavy", i64),
        ("hot_rows", i64),
        ("csl_blocks", i64),
        ("gather_rows", i64),
        ("leaf_blocks", i64),
        ("leaf_blocked_nnz", i64),
        ("leaf_head_share_ppm", i64),
    ]


# (name, argtypes) -- every function returns int status unless listed in _VOID
_SIGS = {
    "hbk_last_error": ([], C.c_char_p),
    "hbk_abi_version": ([], C.c_int),
    "hbk_device_sms": ([C.POINTER(C.c_int)], C.c_int),
    "hbk_coo_create": ([C.c_int, C.POINTER(i64), i64, vp, vp, vp, vp, C.POINTER(vp)], C.c_int),
    "hbk_coo_create_f32": ([C.c_int, C.POINTER(i64), i64, vp, vp, vp, vp, C.POINTER(vp)], C.c_int),
    "hbk_coo_info_get": ([vp, C.POINTER(CooInfo)], C.c_int),
    "hbk_coo_export": ([vp, vp, vp, vp], C.c_int),
    "hbk_coo_device_arrays": ([vp, C.POINTER(vp), C.POINTER(vp)], C.c_int),
    "hbk_coo_export_device": ([vp, vp, vp, vp, vp], C.c_int),
    "hbk_coo_sort": ([vp, vp, vp, C.POINTER(vp)], C.c_int),
    "hbk_coo_canonicalize": ([vp, C.c_int, vp, C.POINTER(vp)], C.c_int),
    "hbk_coo_slices": ([vp, C.c_int, vp, C.POINTER(vp)], C.c_int),
    "hbk_coo_retain": ([vp], None),
    "hbk_coo_release": ([vp], None),
    "hbk_csl_info_get": ([vp, C.POINTER(CslInfo)], C.c_int),
    "hbk_csl_export": ([vp, C.c_int, vp, vp], C.c_int),
    "hbk_csl_retain": ([vp], None),
    "hbk_csl_release": ([vp], None),
    "hbk_csf_info_get": ([vp, C.POINTER(CsfInfo)], C.c_int),
    "hbk_csf_export": ([vp, C.c_int, C.c_int, vp, vp], C.c_int),
    "hbk_build_csf": ([vp, vp, vp, C.POINTER(vp)], C.c_int),
    "hbk_build_hbcsf": ([vp, vp, vp, C.POINTER(vp), C.POINTER(vp), C.POINTER(vp)], C.c_int),
    "hbk_classify_slices": ([vp, vp, vp], C.c_int),
    "hbk_csf_population": ([vp, vp, vp], C.c_int),
    "hbk_split_fibers": ([vp, i64, vp, C.POINTER(vp)], C.c_int),
    "hbk_csf_retain": ([vp], None),
    "hbk_csf_release": ([vp], None),
    "hbk_assign_slice_blocks": ([vp, i64, vp, C.POINTER(vp)], C.c_int),
    "hbk_sched_from_units": ([vp, vp, i64, vp, vp, C.POINTER(vp)], C.c_int),
    "hbk_sched_info_get": ([vp, C.POINTER(SchedInfo)], C.c_int),
    "hbk_sched_export": ([vp, C.c_int, vp, vp], C.c_int),
    "hbk_sched_validate": ([vp, vp, vp], C.c_int),
    "hbk_sched_retain": ([vp], None),
    "hbk_sched_release": ([vp], None),
    "hbk_plan_create": ([vp, vp, vp, vp, C.c_int, C.c_int, vp, C.POINTER(vp)], C.c_int),
    "hbk_plan_info_get": ([vp, C.POINTER(PlanInfo)], C.c_int),
    "hbk_plan_execute": ([vp, vp, vp, vp], C.c_int),
    "hbk_plan_execute_f64": ([vp, vp, vp, vp], C.c_int),
    "hbk_plan_release": ([vp], None),
    "hbk_coo_slice_histogram": ([vp, C.c_int, vp, vp], C.c_int),
    "hbk_coo_fiber_histogram": ([vp, C.c_int, C.c_int, vp, vp], C.c_int),
    "hbk_coo_select_rows": ([vp, C.c_int, i64, i64, vp, C.POINTER(vp)], C.c_int),
    "hbk_coo_shard_rows": ([vp, C.c_int, i64, i64, vp, C.POINTER(vp)], C.c_int),
    "hbk_plan_probe": ([vp, vp, vp], C.c_int),
    "hbk_row_ceiling": ([i64, C.c_int, i64, vp], C.c_int),
    "hbk_row_ceiling_stream": ([vp, i64, i64, C.c_int, vp], C.c_int),
    "hbk_nonfinite_f32": ([vp, vp, C.c_int, vp, vp], C.c_int),
    "hbk_stage_f64_to_f32": ([vp, vp, C.c_int, vp, vp, vp, vp], C.c_int),
    "hbk_stage_f64_to_f64": ([vp, vp, C.c_int, vp, vp, vp, vp], C.c_int),
    "hbk_plan_rows": ([vp, vp, C.POINTER(C.c_int64), vp], C.c_int),
    "hbk_stream_synchronize": ([vp], C.c_int),
    "hbk_plan_execute_ex": ([vp, vp, vp, C.c_int, vp], C.c_int),
    "hbk_als_update_rows": ([vp, vp, C.c_int64, C.c_int, vp, vp, vp, vp, vp, vp], C.c_int),
    "hbk_tns_parse": ([C.c_char_p, i64, C.c_int, vp, C.c_int, C.POINTER(vp)], C.c_int),
    "hbk_tns_load": ([C.c_char_p, C.c_int, vp, C.c_int, C.POINTER(vp)], C.c_int),
    "hbk_tns_info": ([vp, C.POINTER(C.c_int), C.POINTER(i64), vp, C.POINTER(i64)], C.c_int),
    "hbk_tns_export": ([vp, vp, vp], C.c_int),
    "hbk_tns_release": ([vp], None),
    "hbk_tns_format": ([vp, vp, i64, C.c_int, C.c_int, C.POINTER(vp), C.POINTER(i64)], C.c_int),
    "hbk_tns_free_text": ([vp], None),
    "hbk_als_update": ([vp, i64, C.c_int, vp, vp, vp, vp, vp, vp], C.c_int),
}

EXPORTED = tuple(_SIGS)

_lib = None
_lock = threading.Lock()


class NativeUnavailable(RuntimeError):
    """libhbk.so is missing or cannot be loaded (no CPU fallback exists)."""


def load_library(path: str | os.PathLike | None = None) -> C.CDLL:
    """Load libhbk.so and bind every symbol of include/hbk.h (no GPU needed)."""
    global _lib
    with _lock:
        if _lib is not None and path is None:
            return _lib
        p = Path(path) if path is not None else Path(os.environ.get("HBK_LIB", LIB_PATH))
        if not p.exists():
            raise NativeUnavailable(
                f"{p} not found: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
            )
        lib = C.CDLL(str(p))
        for name, (args, res) in _SIGS.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = res
        if lib.hbk_abi_version() != 1:
            raise NativeUnavailable("libhbk ABI version mismatch")
        if path is None:
            _lib = lib
        return lib


def lib() -> C.CDLL:
    return _lib if _lib is not None else load_library()


def check(status: int) -> None:
    """Map an hbk status to the reference's exception types."""
    if status == HBK_OK:
        return
    msg = lib().hbk_last_error().decode(errors="replace")
    if status == HBK_EINVAL:
        raise ValueError(msg)
    if status == HBK_ETYPE:
        raise TypeError(msg)
    if status == HBK_ENOMEM:
        raise MemoryError(msg)
    raise RuntimeError(msg)


def call(name: str, *args) -> None:
    check(getattr(lib(), name)(*args))


_device_checked = False


def require_device():
    """Import torch and make sure a CUDA device is present; fail loudly."""
    global _device_checked
    import torch

    if not _device_checked:
        if not torch.cuda.is_available():
            raise NativeUnavailable(
                "no CUDA device: the HB-CSF kernels run only on the GPU (no CPU fallback)"
            )
        lib()
        _device_checked = True
    return torch


def stream_ptr():
    """cudaStream_t of torch's current stream on the current device (the
    raw-stream accessor: torch.cuda.current_stream() costs ~15 us of Python
    per call, a measurable share of a small host-array MTTKRP call)."""
    torch = require_device()
    raw = getattr(torch._C, "_cuda_getCurrentRawStream", None)
    if raw is not None:
        return C.c_void_p(raw(torch._C._cuda_getDevice()))
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


class Handle:
    """Owns one reference to a native object; releases it on collection."""

    __slots__ = ("ptr", "_release", "__weakref__")

    def __init__(self, ptr, release: str):
        if not ptr:
            raise RuntimeError("null native handle")
        self.ptr = C.c_void_p(ptr if isinstance(ptr, int) else ptr.value)
        self._release = release

    def __del__(self):
        try:
            if self.ptr and _lib is not None:
                getattr(_lib, self._release)(self.ptr)
                self.ptr = None
        except Exception:
            pass


def new_out() -> C.c_void_p:
    return C.c_void_p()


def i64_array(values) -> C.Array:
    vals = [int(v) for v in values]
    return (i64 * max(1, len(vals)))(*vals)


def int_array(values) -> C.Array:
    vals = [int(v) for v in values]
    return (C.c_int * max(1, len(vals)))(*vals)
