"""MTTKRP over each storage format, on the GPU.

Mirrors ``tenkit.kernels`` (pkg/src/tenkit/kernels.py): same function names,
signatures, argument checks, exceptions and ``OpCount`` integers.  Every call
runs libhbk's sm_100a kernel (one persistent launch per call; see
csrc/mttkrp.cu).  There is no CPU path: without libhbk.so or a CUDA device
the calls raise.

Factor matrices may be NumPy arrays (the reference's calling convention:
uploaded as fp32, result returned as a float64 ``np.ndarray``) or CUDA
tensors (fp32, row-major; the result is then a CUDA fp32 tensor and nothing
leaves the device).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Sequence

import numpy as np

from . import _native as N
from .coo import CooTensor
from .formats import CslSlices, CsfTensor, HbCsfTensor

Factors = Sequence


@dataclass(frozen=True)
class OpCount:
    """Floating-point multiply and add counts (kernels.py:44-59)."""

    muls: int
    adds: int

    @property
    def total(self) -> int:
        return self.muls + self.adds

    def __add__(self, other: "OpCount") -> "OpCount":
        return OpCount(self.muls + other.muls, self.adds + other.adds)

    def to_dict(self) -> dict:
        return {"muls": self.muls, "adds": self.adds, "total": self.total}


def _is_device(f) -> bool:
    return type(f).__module__.startswith("torch") and getattr(f, "is_cuda", False)


def _check_factors(dims: tuple[int, ...], factors: Factors, mode: int, check_finite: bool = True) -> int:
    """Validate factor shapes against dims; factors[mode] is not inspected
    (kernels.py:62-88).  Returns the shared rank R."""
    if not 0 <= mode < len(dims):
        raise ValueError(f"mode {mode} out of range for order {len(dims)}")
    if len(factors) != len(dims):
        raise ValueError(f"expected {len(dims)} factor matrices, got {len(factors)}")
    rank = None
    for d, f in enumerate(factors):
        if d == mode:
            continue
        if _is_device(f):
            shape = tuple(f.shape)
            finite = (lambda f=f: bool(f.isfinite().all()))
        else:
            f = np.asarray(f)
            shape = f.shape
            finite = (lambda f=f: bool(np.isfinite(f).all()))
        if len(shape) != 2 or shape[0] != dims[d]:
            raise ValueError(f"factor {d} must have shape ({dims[d]}, R), got {shape}")
        if rank is None:
            rank = int(shape[1])
        elif shape[1] != rank:
            raise ValueError("factor matrices disagree on rank")
        # host arrays under "staged": checked while they are converted into
        # the pinned upload buffers (_HostStage.upload), before any kernel runs
        if check_finite and not (check_finite == "staged" and not _is_device(f)) and not finite():
            raise ValueError(f"factor {d} has non-finite entries")
    assert rank is not None
    return rank


class _HostStage:
    """Upload/download path of the host-array calling convention (the
    reference's: NumPy float64 factors in, NumPy float64 rows out).

    NumPy float64 factors go through libhbk's native staging
    (hbk_stage_f64_to_f32 / _f64): a pool of host threads converts them into
    page-locked buffers with streaming stores and the host-to-device copies
    follow chunk by chunk, with the non-finite check of kernels.py:82-86
    done on the way (raised before any kernel runs).  Page-locked torch
    tensors of the kernel dtype are copied as they are and checked on the
    device (one hbk_nonfinite_f32 launch after the MTTKRP, flags returned with
    the rows); other host arrays (other dtypes) are converted on a Python
    thread pool and checked the same way.  When a check fires, the host
    source tells a non-finite entry from a finite one beyond the float32
    range.  The rows come back widened to float64 on the device, through one
    async copy into page-locked memory that becomes the returned array."""

    CHUNK_BYTES = 1 << 20  # conversion work unit (bytes of the source factor)

    def __init__(self):
        import os
        import threading
        from concurrent.futures import ThreadPoolExecutor

        self.lock = threading.Lock()
        self.workers = max(1, min(16, (os.cpu_count() or 1)))
        self.pool = ThreadPoolExecutor(self.workers, thread_name_prefix="hbk-stage")
        self.bufs = {}

    def _pinned(self, torch, key, n, dtype):
        buf, ev = self.bufs.get(key, (None, None))
        if buf is None or buf.numel() < n or buf.dtype != dtype:
            buf, ev = torch.empty(max(n, 1), dtype=dtype, pin_memory=True), None
        if ev is not None:
            ev.synchronize()  # the previous copy out of this buffer is done
        return buf

    def _spans(self, rows, width, itemsize):
        step = max(1, self.CHUNK_BYTES // max(1, width * itemsize))
        return [(a, min(rows, a + step)) for a in range(0, rows, step)]

    def _map(self, fn, spans):
        if len(spans) == 1:
            return [fn(*spans[0])]
        return [fu.result() for fu in [self.pool.submit(fn, a, b) for a, b in spans]]

    def upload_all(self, torch, items, dt):
        """items: [(d, host array)] -> ({d: CUDA tensor}, deferred checks).
        Every uploaded copy is returned in ``checks`` as (d, device tensor,
        host source) for the device finiteness scan after the launch.
        Page-locked torch tensors of the kernel dtype are copied as they are.
        Other factors are
        converted concurrently (one pool task per factor, or per chunk of a
        large one); the host-to-device copies are issued by the calling
        thread, on its current stream, as soon as each factor is staged."""
        srcs = {}
        out, checks = {}, []
        for d, f in items:
            if _is_pinned_tensor(f, dt):
                # page-locked host tensor of the kernel dtype: one async copy,
                # finiteness checked on the device after the launch
                dev = torch.empty(tuple(f.shape), dtype=dt, device="cuda")
                dev.copy_(f, non_blocking=True)
                out[d] = dev
                checks.append((d, dev, None))  # checked after the launch (_finish)
                continue
            src = np.ascontiguousarray(f)
            if src.ndim != 2:
                raise ValueError(f"factor {d} must be a 2-D array")
            srcs[d] = src
        # float64 -> fp32 (the reference convention) or -> fp64 (precision=
        # "fp64"): narrowed / copied by libhbk's host threads with streaming
        # stores and sent chunk by chunk as it goes (hbk_stage_f64_to_f32/_f64)
        nat = [d for d, s in srcs.items()
               if dt in (torch.float32, torch.float64) and s.dtype == np.float64]
        fn = "hbk_stage_f64_to_f32" if dt == torch.float32 else "hbk_stage_f64_to_f64"
        if nat:
            with self.lock:
                stages, devs = {}, {}
                for d in nat:
                    rows, width = srcs[d].shape
                    stages[d] = self._pinned(torch, ("in", d), rows * width, dt)
                    devs[d] = torch.empty((rows, width), dtype=dt, device="cuda")
                k = len(nat)
                flags = (C.c_int32 * k)()
                N.call(fn,
                       (C.c_void_p * k)(*[srcs[d].ctypes.data for d in nat]),
                       (C.c_int64 * k)(*[srcs[d].size for d in nat]), k,
                       (C.c_void_p * k)(*[stages[d].data_ptr() for d in nat]),
                       (C.c_void_p * k)(*[devs[d].data_ptr() for d in nat]),
                       flags, N.stream_ptr())
                ev = torch.cuda.Event()
                ev.record(torch.cuda.current_stream())
                for i, d in enumerate(nat):
                    self.bufs[("in", d)] = (stages[d], ev)
                    if flags[i]:
                        _raise_nonfinite(d, srcs[d])
                    out[d] = devs[d]
                    del srcs[d]
        with self.lock:
            stages, jobs = {}, []
            for d, src in srcs.items():
                rows, width = src.shape
                buf = self._pinned(torch, ("in", d), rows * width, dt)
                stages[d] = (buf, buf.numpy()[: rows * width].reshape(rows, width))
                for a, b in self._spans(rows, width, src.itemsize):
                    jobs.append((d, a, b))
            if not jobs:
                return out, checks

            def convert(d, a, b):
                with np.errstate(over="ignore", invalid="ignore"):  # reported by the device scan
                    np.copyto(stages[d][1][a:b], srcs[d][a:b], casting="unsafe")

            if len(jobs) == 1:
                futs = [None]
                convert(*jobs[0])
            else:
                futs = [self.pool.submit(convert, *j) for j in jobs]
            left = {d: sum(1 for j in jobs if j[0] == d) for d in srcs}
            for i, (d, a, b) in enumerate(jobs):
                if futs[i] is not None:
                    futs[i].result()
                left[d] -= 1
                if left[d] == 0:
                    rows, width = srcs[d].shape
                    dev = torch.empty((rows, width), dtype=dt, device="cuda")
                    if rows * width:
                        dev.copy_(stages[d][0][: rows * width].view(rows, width), non_blocking=True)
                    out[d] = dev
                    checks.append((d, dev, srcs[d]))
            ev = torch.cuda.Event()
            ev.record(torch.cuda.current_stream())
            for d in srcs:
                self.bufs[("in", d)] = (stages[d][0], ev)
        return out, checks

    # outputs up to this size are widened on the device and copied straight
    # into a page-locked float64 array (torch's caching host allocator) that
    # is returned as the NumPy result; larger ones come back as fp32 into a
    # reused pinned buffer and are widened on host threads
    PINNED_OUT_BYTES = 256 << 20

    def download(self, torch, y, flags=None):
        """Device rows -> NumPy float64 rows (+ the host copy of the device
        int32 ``flags`` vector, read back under the same synchronisation)."""
        n = y.numel()
        with self.lock:
            fbuf = None
            if flags is not None and flags.numel():
                fbuf = self._pinned(torch, ("flags",), flags.numel(), flags.dtype)
                fbuf[: flags.numel()].copy_(flags, non_blocking=True)
            if n * 8 <= self.PINNED_OUT_BYTES:
                host = torch.empty(tuple(y.shape), dtype=torch.float64, pin_memory=n > 0)
                if n:
                    host.copy_(y if y.dtype == torch.float64 else y.to(torch.float64),
                               non_blocking=True)
                N.call("hbk_stream_synchronize", N.stream_ptr())
                out = host.numpy()
            else:
                out = np.empty(tuple(y.shape), dtype=np.float64)
                rows = int(y.shape[0])
                width = n // max(1, rows)
                buf = self._pinned(torch, ("out",), n, y.dtype)
                buf[:n].view(y.shape).copy_(y, non_blocking=True)
                N.call("hbk_stream_synchronize", N.stream_ptr())
                src = buf.numpy()[:n].reshape(rows, width)
                dst = out.reshape(rows, width)
                step = max(1, (2 << 20) // max(1, width * 8))
                spans = [(a, min(rows, a + step)) for a in range(0, rows, step)]
                self._map(lambda a, b: np.copyto(dst[a:b], src[a:b]), spans)
                self.bufs[("out",)] = (buf, None)
            fl = fbuf[: flags.numel()].tolist() if fbuf is not None else []
        return out, fl


_stage = None


def _is_pinned_tensor(f, dt) -> bool:
    return (type(f).__module__.startswith("torch") and not getattr(f, "is_cuda", True)
            and f.dtype == dt and f.is_contiguous() and f.dim() == 2 and f.is_pinned())


def _host_stage() -> _HostStage:
    global _stage
    if _stage is None:
        _stage = _HostStage()
    return _stage


def _device_factors(factors: Factors, mode: int, precision: str = "fp32"):
    """Contiguous CUDA copies/views (fp32, or fp64 for precision="fp64") of the
    non-mode factors + the pointer array.  Host arrays go through the pinned
    staging path (and are checked for non-finite entries there)."""
    torch = N.require_device()
    dt = torch.float64 if precision == "fp64" else torch.float32
    keep = []
    ptrs = (C.c_void_p * len(factors))()
    host = [(d, f) for d, f in enumerate(factors) if d != mode and not _is_device(f)]
    staged, checks = _host_stage().upload_all(torch, host, dt) if host else ({}, [])
    on_device = not host
    for d, f in enumerate(factors):
        if d == mode:
            ptrs[d] = None
            continue
        t = staged.get(d)
        if t is None:
            t = f if (f.dtype == dt and f.is_contiguous()) else f.to(dt).contiguous()
        if t.data_ptr() % 16:
            t = t.clone()
        keep.append(t)
        ptrs[d] = t.data_ptr()
    return ptrs, keep, on_device, checks


class _Plan:
    """A libhbk plan (work list for one mode/rank/bucket set) plus its info."""

    __slots__ = ("h", "info", "rows", "rank", "_owned")

    def __init__(self, coo, csl, csf, sched, mode: int, rank: int, rows: int):
        out = N.new_out()
        N.call("hbk_plan_create", coo, csl, csf, sched, int(mode), int(rank), N.stream_ptr(),
               C.byref(out))
        self.h = N.Handle(out, "hbk_plan_release")
        info = N.PlanInfo()
        N.call("hbk_plan_info_get", self.h.ptr, C.byref(info))
        self.info = info
        self.rows = rows
        self.rank = rank
        self._owned = None

    @property
    def opcount(self) -> OpCount:
        return OpCount(int(self.info.op_muls), int(self.info.op_adds))

    def owned_rows(self):
        """Device int32 tensor of the output rows the buckets own, ascending
        (hbk_plan_rows); rows outside it are zero in every MTTKRP result."""
        if self._owned is None:
            torch = N.require_device()
            n = C.c_int64(0)
            N.call("hbk_plan_rows", self.h.ptr, None, C.byref(n), N.stream_ptr())
            out = torch.empty(max(1, n.value), dtype=torch.int32, device="cuda")
            N.call("hbk_plan_rows", self.h.ptr, C.c_void_p(out.data_ptr()), C.byref(n),
                   N.stream_ptr())
            self._owned = out[: n.value]
        return self._owned

    def probe(self, factor_ptrs) -> None:
        """Launch the plan's gather-only calibration kernels (hbk_plan_probe)."""
        N.call("hbk_plan_probe", self.h.ptr, factor_ptrs, N.stream_ptr())

    def execute(self, factor_ptrs, out=None, precision: str = "fp32", skip_unowned: bool = False):
        """skip_unowned: rows no bucket owns may be left unwritten (fp32 fast
        path; callers that read only owned_rows())."""
        torch = N.require_device()
        dt = torch.float64 if precision == "fp64" else torch.float32
        if out is None:
            out = torch.empty((self.rows, self.rank), dtype=dt, device="cuda")
        if precision == "fp64":
            N.call("hbk_plan_execute_f64", self.h.ptr, factor_ptrs, C.c_void_p(out.data_ptr()),
                   N.stream_ptr())
        else:
            N.call("hbk_plan_execute_ex", self.h.ptr, factor_ptrs, C.c_void_p(out.data_ptr()),
                   1 if skip_unowned else 0, N.stream_ptr())
        return out


def _get_plan(owner, key, build):
    plan = owner._plans.get(key)
    if plan is None:
        plan = build()
        owner._plans[key] = plan
    return plan


def _check_precision(precision: str) -> str:
    if precision not in ("fp32", "fp64"):
        raise ValueError(f"precision must be 'fp32' or 'fp64', got {precision!r}")
    return precision


def _nonfinite_flags(torch, tensors):
    """Device int32 vector: 1 where the tensor holds a NaN/Inf (fp32 tensors:
    one hbk_nonfinite_f32 launch over all of them)."""
    flags = torch.empty(len(tensors), dtype=torch.int32, device="cuda")
    if all(t.dtype == torch.float32 for t in tensors) and len(tensors) <= 8:
        ptrs = (C.c_void_p * len(tensors))(*[t.data_ptr() for t in tensors])
        counts = (C.c_int64 * len(tensors))(*[t.numel() for t in tensors])
        N.call("hbk_nonfinite_f32", ptrs, counts, len(tensors), C.c_void_p(flags.data_ptr()),
               N.stream_ptr())
    else:
        for i, t in enumerate(tensors):
            flags[i] = (~torch.isfinite(t)).any().to(torch.int32)
    return flags


def _finish(plan: _Plan, factors, mode: int, out=None, precision: str = "fp32"):
    ptrs, keep, on_device, checks = _device_factors(factors, mode, _check_precision(precision))
    y = plan.execute(ptrs, out, precision)
    if on_device:
        return y, plan.opcount
    torch = N.require_device()
    # pinned host tensors are checked on the device (one hbk_nonfinite_f32
    # launch), after the MTTKRP launch so it does not wait for the scan; the
    # flags come back with the rows
    flags = _nonfinite_flags(torch, [dev for _, dev, _ in checks]) if checks else None
    rows, bad = _host_stage().download(torch, y, flags)
    for (d, _, src), b in sorted(zip(checks, bad), key=lambda x: x[0][0]):
        if b:
            _raise_nonfinite(d, src)
    return rows, plan.opcount


def _raise_nonfinite(d: int, src) -> None:
    """The fp32 copy of factor d holds a NaN/Inf: a non-finite source entry
    (kernels.py:82-86) or a finite float64 beyond the float32 range."""
    if src is not None and np.isfinite(src).all():
        raise ValueError(f"factor {d} has entries outside the float32 range of the fp32 "
                         "kernel; pass precision='fp64'")
    raise ValueError(f"factor {d} has non-finite entries")


def plan_for(rep, mode: int, rank: int, schedule=None) -> _Plan:
    """The cached libhbk plan that ``mttkrp(rep, ..., mode)`` executes."""
    dims = rep.dims
    if isinstance(rep, HbCsfTensor):
        sh = schedule._device_for(rep.csf_part) if schedule is not None else None
        key = (mode, rank, None if sh is None else sh.ptr.value)
        return _get_plan(rep, key, lambda: _Plan(
            rep.coo_part._dev().ptr if rep.coo_part.nnz else None,
            rep.csl_part._h.ptr, rep.csf_part._h.ptr, None if sh is None else sh.ptr,
            mode, rank, dims[mode]))
    if isinstance(rep, CsfTensor):
        sh = schedule._device_for(rep) if schedule is not None else None
        key = (mode, rank, None if sh is None else sh.ptr.value)
        return _get_plan(rep, key, lambda: _Plan(None, None, rep._h.ptr,
                                                 None if sh is None else sh.ptr, mode, rank,
                                                 dims[mode]))
    if isinstance(rep, CslSlices):
        return _get_plan(rep, (mode, rank, None),
                         lambda: _Plan(None, rep._h.ptr, None, None, mode, rank, dims[mode]))
    if isinstance(rep, CooTensor):
        return _get_plan(rep, (mode, rank, None),
                         lambda: _Plan(None, rep._slices(mode).ptr, None, None, mode, rank, dims[mode]))
    raise TypeError(f"no MTTKRP kernel for {type(rep).__name__}")


def mttkrp_coo(t: CooTensor, factors: Factors, mode: int, threads: int = 1, *, precision: str = "fp32"):
    """MTTKRP over a coordinate list (kernels.py:109-151).

    The entries are grouped by their mode-``mode`` coordinate on the GPU
    (sorted under (mode, *rest) unless already mode-major) and reduced per
    output row; ``threads`` is accepted for API compatibility."""
    r = _check_factors(t.dims, factors, mode, check_finite="staged")
    return _finish(plan_for(t, mode, r), factors, mode, precision=precision)


def mttkrp_csf(c: CsfTensor, factors: Factors, mode: int, *, precision: str = "fp32"):
    """MTTKRP over a CSF tree built with mode_order[0] == mode (kernels.py:154-186)."""
    if c.mode_order[0] != mode:
        raise ValueError(f"tree was built for mode {c.mode_order[0]}, asked for mode {mode}")
    r = _check_factors(c.dims, factors, mode, check_finite="staged")
    return _finish(plan_for(c, mode, r), factors, mode, precision=precision)


def mttkrp_csl(s: CslSlices, factors: Factors, mode: int, threads: int = 1, *,
               precision: str = "fp32"):
    """MTTKRP over compressed slices (kernels.py:189-226)."""
    if s.mode_order[0] != mode:
        raise ValueError(f"slices were built for mode {s.mode_order[0]}, asked for mode {mode}")
    r = _check_factors(s.dims, factors, mode, check_finite="staged")
    return _finish(plan_for(s, mode, r), factors, mode, precision=precision)


def mttkrp_hbcsf(h: HbCsfTensor, factors: Factors, mode: int, schedule=None, threads: int = 1, *,
                 precision: str = "fp32"):
    """MTTKRP over the hybrid format, all three buckets in one launch
    (kernels.py:229-253).  A schedule applies to the CSF bucket only."""
    if h.mode_order[0] != mode:
        raise ValueError(f"hybrid was built for mode {h.mode_order[0]}, asked for mode {mode}")
    if schedule is not None:
        schedule.validate_for(h.csf_part)
    r = _check_factors(h.dims, factors, mode, check_finite="staged")
    return _finish(plan_for(h, mode, r, schedule), factors, mode, precision=precision)


def mttkrp_scheduled(c: CsfTensor, schedule, factors: Factors, mode: int, threads: int = 1, *,
                     precision: str = "fp32"):
    """MTTKRP over a CSF tree driven by a block schedule (kernels.py:256-342):
    one device work unit per schedule unit."""
    if c.mode_order[0] != mode:
        raise ValueError(f"tree was built for mode {c.mode_order[0]}, asked for mode {mode}")
    schedule.validate_for(c)
    r = _check_factors(c.dims, factors, mode, check_finite="staged")
    return _finish(plan_for(c, mode, r, schedule), factors, mode, precision=precision)


def mttkrp(rep, factors: Factors, mode: int, **kwargs):
    """Dispatch MTTKRP by representation type (kernels.py:345-355)."""
    if isinstance(rep, CooTensor):
        return mttkrp_coo(rep, factors, mode, **kwargs)
    if isinstance(rep, CsfTensor):
        return mttkrp_csf(rep, factors, mode, **kwargs)
    if isinstance(rep, CslSlices):
        return mttkrp_csl(rep, factors, mode, **kwargs)
    if isinstance(rep, HbCsfTensor):
        return mttkrp_hbcsf(rep, factors, mode, **kwargs)
    raise TypeError(f"no MTTKRP kernel for {type(rep).__name__}")


def mttkrp_device(rep, factors, mode: int, out=None, schedule=None, precision: str | None = None,
                  skip_unowned: bool = False):
    """Device fast path: CUDA factors in, CUDA (dims[mode], R) out, no host
    synchronisation and no finiteness scan.  The kernel precision follows the
    factors' dtype (float64 -> fp64 kernel) unless given.  Returns (out, OpCount)."""
    if getattr(rep, "mode_order", None) is not None and rep.mode_order[0] != mode:
        raise ValueError(f"representation was built for mode {rep.mode_order[0]}, asked for mode {mode}")
    r = _check_factors(rep.dims, factors, mode, check_finite=False)
    if precision is None:
        ref = next(f for d, f in enumerate(factors) if d != mode)
        precision = "fp64" if str(getattr(ref, "dtype", "")) == "torch.float64" else "fp32"
    plan = plan_for(rep, mode, r, schedule)
    ptrs, keep, _, _ = _device_factors(factors, mode, _check_precision(precision))
    return plan.execute(ptrs, out, precision, skip_unowned), plan.opcount
