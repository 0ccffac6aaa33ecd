"""Row-sharded multi-GPU CP-ALS (config 5 of BASELINE.json).

One process per GPU (torchrun), ``torch.distributed`` for the plumbing
(NCCL on the GPUs, gloo for the CPU tests).  The algorithm is the reference's
``cp_als`` (cpd.py:198-271) with every mode's rows partitioned:

* mode n's output rows are cut into contiguous ranges balanced by nonzero
  count (``shard.plan_row_ranges``); rank g owns rows [lo_g, hi_g) of
  factor n and builds the HB-CSF of the entries in that range only
  (``hbk_coo_shard_rows``: rebased, so its MTTKRP writes exactly those rows);
* the MTTKRP of a mode needs no communication (slices are independent,
  kernels.py:154-186);
* the ALS update ``F_n[rows_g] = Y_g · V†`` is row-local (cpd.py:170-172), V
  is built from Grams every rank holds;
* exchanges per mode: one all-gather of the fp32 rows the MTTKRP kernels read
  (uneven shards padded), one all-reduce of the R×R fp64 Gram partials
  (cpd.py:39-42), one all-reduce of the finiteness flag; per sweep one scalar
  all-reduce for ⟨X, X̂⟩ (cpd.py:176-184).
* fp64 master rows stay on their owner; column norms for the normalisation
  (cpd.py:187-195) come from the diagonal of the all-reduced Gram, so every
  rank applies identical scalings.  The full fp64 factors are gathered once,
  at the end, for the returned KruskalModel.
"""
from __future__ import annotations

import math
import time
import warnings

import numpy as np

from .coo import CooTensor, allmode_order, canonicalize
from .cpd import AlsIteration, KruskalModel, NumericalError, hadamard_all_but, pinv_spsd
from .shard import plan_row_ranges


def _dist():
    import torch.distributed as dist

    if not dist.is_available() or not dist.is_initialized():
        raise RuntimeError("cp_als_distributed needs an initialised torch.distributed process group")
    return dist


def allgather_padded(torch, dist, local, ranges, group=None):
    """Replicate a row-sharded (rows, R) matrix: one all_gather_into_tensor of
    max-shard-sized buffers, then the padding is dropped."""
    world = len(ranges)
    width = local.shape[1]
    cap = max(1, max(hi - lo for lo, hi in ranges))
    buf = torch.zeros((cap, width), dtype=local.dtype, device=local.device)
    buf[: local.shape[0]] = local
    out = torch.empty((world * cap, width), dtype=local.dtype, device=local.device)
    if hasattr(dist, "all_gather_into_tensor") and local.device.type == "cuda":
        dist.all_gather_into_tensor(out, buf, group=group)
    else:
        dist.all_gather(list(out.chunk(world)), buf, group=group)
    return torch.cat([out[g * cap: g * cap + (hi - lo)] for g, (lo, hi) in enumerate(ranges)])


class DeviceShards:
    """Per-mode HB-CSF of this rank's row range, MTTKRP on the GPU."""

    def __init__(self, t: CooTensor, world: int, me: int):
        from . import shard
        from .formats import build_hbcsf

        self.me = me
        self.ranges, self.reps = [], []
        for mode in range(t.order):
            hist = shard.slice_histogram(t, mode).cpu().numpy()
            ranges = plan_row_ranges(hist, world)
            lo, hi = ranges[me]
            self.ranges.append(ranges)
            if hi > lo:
                part = shard.shard_rows(t, mode, lo, hi)
                self.reps.append(build_hbcsf(part, allmode_order(t.dims, mode)))
            else:
                self.reps.append(None)

    def __call__(self, mode: int, factors32):
        from .kernels import mttkrp_device

        lo, hi = self.ranges[mode][self.me]
        rep = self.reps[mode]
        ref = factors32[(mode + 1) % len(factors32)]
        if rep is None:
            return ref.new_zeros((0, ref.shape[1]))
        fs = list(factors32)
        fs[mode] = factors32[mode][: hi - lo]  # shape only; factors[mode] is not read
        y, _ = mttkrp_device(rep, fs, mode)
        return y


def cp_als_distributed(t: CooTensor, rank: int = 32, max_iters: int = 50, fit_tol: float = 1e-8,
                       seed: int = 0, *, group=None, local_mttkrp=None, ranges=None,
                       device=None):
    """CP-ALS over ``world`` processes, each owning a row range of every mode.

    Every rank passes the same tensor ``t`` (it is canonicalised and sharded
    locally).  Returns the same (KruskalModel, [AlsIteration]) as ``cp_als`` on
    every rank.  ``local_mttkrp(mode, factors32) -> (rows_g, R)`` and
    ``ranges`` (per mode, the row ranges of all ranks) replace the GPU shards
    (used by the CPU tests); by default the HB-CSF shards are built on the GPU
    and the collectives run on NCCL."""
    import torch

    dist = _dist()
    world = dist.get_world_size(group)
    me = dist.get_rank(group)
    if rank < 1:
        raise ValueError("rank must be at least 1")
    if max_iters < 0:
        raise ValueError("max_iters must be nonnegative")
    if local_mttkrp is None:
        from . import _native as N

        N.require_device()
        device = torch.device("cuda", torch.cuda.current_device())
        t = canonicalize(t)
        if t.nnz == 0:
            raise ValueError("cannot decompose an empty tensor")
        shards = DeviceShards(t, world, me)
        ranges = shards.ranges
        local_mttkrp = shards
    else:
        device = torch.device(device or "cpu")
        if ranges is None:
            raise ValueError("ranges are required with a custom local_mttkrp")
    dims = t.dims
    order = len(dims)
    over = [d for d, dim in enumerate(dims) if rank > dim]
    if over:
        warnings.warn(f"rank {rank} exceeds the extent of mode(s) {over}; the problem is "
                      "over-complete and factors will be rank-deficient", RuntimeWarning)

    rng = np.random.default_rng(seed)
    init = [rng.random((dim, rank)) for dim in dims]  # cpd.py:231-232, identical on every rank
    own = [ranges[d][me] for d in range(order)]
    f64 = [torch.from_numpy(init[d][lo:hi].copy()).to(device) for d, (lo, hi) in enumerate(own)]
    f32 = [torch.from_numpy(init[d]).to(device=device, dtype=torch.float32) for d in range(order)]

    def gram_allreduce(local):
        g = local.T @ local
        dist.all_reduce(g, group=group)
        g = g.cpu().numpy()
        return (g + g.T) * 0.5

    def scalar_allreduce(x):
        v = torch.tensor([x], dtype=torch.float64, device=device)
        dist.all_reduce(v, group=group)
        return float(v.item())

    def all_true(flag):
        v = torch.tensor([0.0 if flag else 1.0], dtype=torch.float64, device=device)
        dist.all_reduce(v, group=group)
        return float(v.item()) == 0.0

    def sync():
        if device.type == "cuda":
            torch.cuda.synchronize(device)

    grams = [gram_allreduce(f) for f in f64]
    norm_x = _value_norm(torch, t)
    last = order - 1

    def fit_of(y_local, grams):
        norm_hat_sq = float((hadamard_all_but(grams, last) * grams[last]).sum())
        inner = scalar_allreduce(float((y_local.double() * f64[last]).sum()))
        err_sq = max(norm_x * norm_x + norm_hat_sq - 2.0 * inner, 0.0)
        return 1.0 - math.sqrt(err_sq) / norm_x

    fit = fit_of(local_mttkrp(last, f32), grams)
    history = [AlsIteration(0, fit, 0.0, (), ())]
    lam = None
    for it in range(1, max_iters + 1):
        seconds = []
        y = None
        for mode in range(order):
            sync()
            tic = time.perf_counter()
            y = local_mttkrp(mode, f32).double()
            vinv = torch.from_numpy(pinv_spsd(hadamard_all_but(grams, mode))).to(device)
            factor = y @ vinv
            if not all_true(bool(torch.isfinite(factor).all())):
                raise NumericalError(f"non-finite factor for mode {mode} in ALS sweep {it}", iteration=it)
            f64[mode] = factor
            f32[mode] = allgather_padded(torch, dist, factor.float(), ranges[mode], group)
            grams[mode] = gram_allreduce(factor)
            sync()
            seconds.append(time.perf_counter() - tic)
        new_fit = fit_of(y, grams)
        lam = _normalize(torch, f64, f32, grams, device)
        if not math.isfinite(new_fit):
            raise NumericalError(f"non-finite fit in ALS sweep {it}", iteration=it)
        delta = new_fit - history[-1].fit
        history.append(AlsIteration(it, new_fit, delta, tuple(seconds), ()))
        if abs(delta) < fit_tol:
            break
    if len(history) == 1:
        lam = _normalize(torch, f64, f32, grams, device)
    full = [allgather_padded(torch, dist, f64[d], ranges[d], group).cpu().numpy() for d in range(order)]
    return KruskalModel(lam=lam, factors=tuple(full)), history


def _value_norm(torch, t: CooTensor) -> float:
    """‖X‖_F (cpd.py:233), on the device when the tensor lives there."""
    if getattr(t, "_values", None) is None and getattr(t, "_handle", None) is not None:
        import ctypes as C

        from . import _native as N

        v = torch.empty(t.nnz, dtype=torch.float64, device="cuda")
        N.call("hbk_coo_export_device", t._dev().ptr, None, C.c_void_p(v.data_ptr()), None,
               N.stream_ptr())
        return float(torch.linalg.vector_norm(v).item())
    return float(np.linalg.norm(t.values))


def _normalize(torch, f64, f32, grams, device):
    """Column norms from diag(G) of the all-reduced Grams (cpd.py:187-195)."""
    lam = None
    for d in range(len(f64)):
        n = np.sqrt(np.maximum(np.diag(grams[d]), 0.0))
        n = np.where(n > 0.0, n, 1.0)
        nt = torch.from_numpy(n).to(device)
        f64[d] = f64[d] / nt
        f32[d] = (f32[d].double() / nt).float()
        grams[d] = grams[d] / np.outer(n, n)
        lam = n.copy() if lam is None else lam * n
    return lam
