"""Row-sharded multi-GPU CP-ALS (config 5 of BASELINE.json).

One process per GPU (torchrun), ``torch.distributed`` for the plumbing
(NCCL on the GPUs, gloo for the CPU tests).  The algorithm is the reference's
``cp_als`` (cpd.py:198-271) with every mode's rows partitioned:

* mode n's output rows are cut into contiguous ranges balanced by cost —
  nonzeros + fibers + a per-row charge (``shard.partition_costs``,
  ``shard.plan_row_ranges``); rank g owns rows [lo_g, hi_g) of
  factor n and builds the HB-CSF of the entries in that range only
  (``hbk_coo_shard_rows``: rebased, so its MTTKRP writes exactly those rows);
* the MTTKRP of a mode needs no communication (slices are independent,
  kernels.py:154-186);
* the ALS update ``F_n[rows_g] = Y_g · V†`` is row-local (cpd.py:170-172) and
  runs fused with the Gram partial and the fit term (``hbk_als_update``);
  V is built from Grams every rank holds;
* exchanges per mode: the touched-rows exchange — each rank receives, in one
  all_to_all, only the rows of the new factor that its own shards of the
  other modes read (``RowExchange``; index lists agreed once) — or, with
  ``exchange="full"``, every rank broadcasts its contiguous fp32 rows into
  every replicated copy; one all-reduce of the R×R fp64 Gram partial
  (cpd.py:39-42); per sweep one scalar all-reduce for ⟨X, X̂⟩ (cpd.py:176-184).
* column normalisation (cpd.py:187-195) is kept as per-column scales folded
  into the next update matrix, so it costs no pass over the factors.
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


def allgather_rows(torch, dist, local, ranges, group=None):
    """Replicate a row-sharded (rows, R) matrix whose ranks own contiguous,
    unequal row ranges (SURVEY §8e "allgatherv = one broadcast per rank"):
    rank r's rows are broadcast from r straight into their place in the full
    matrix, so every rank receives exactly the rows it does not own — no
    padding to the largest range (the cost-balanced cuts give ranges of very
    different sizes: 24M of flickr-3d mode 1's 28M rows on one of 8 ranks)."""
    me = dist.get_rank(group)
    width = local.shape[1]
    total = ranges[-1][1] if ranges else 0
    out = torch.empty((total, width), dtype=local.dtype, device=local.device)
    lo, hi = ranges[me]
    out[lo:hi] = local[: hi - lo]
    works = []
    for r, (a, b) in enumerate(ranges):
        if b > a:
            src = dist.get_global_rank(group, r) if group is not None else r
            works.append(dist.broadcast(out[a:b], src=src, group=group, async_op=True))
    for w in works:
        w.wait()
    return out


class DeviceShards:
    """Per-mode HB-CSF of this rank's row range, MTTKRP on the GPU, and the
    factor rows those shards reference (for the touched-rows exchange)."""

    def __init__(self, t: CooTensor, world: int, me: int):
        import ctypes as C

        import torch

        from . import _native as N
        from . import shard
        from .formats import build_hbcsf

        self.me = me
        self.ranges, self.reps = [], []
        refs = [[] for _ in range(t.order)]
        # needed_by[mode][d]: rows of factor d this rank's shard of `mode` reads
        self.needed_by = [[None] * t.order for _ in range(t.order)]
        for mode in range(t.order):
            ranges = plan_row_ranges(shard.partition_costs(t, mode).cpu().numpy(), world)
            lo, hi = ranges[me]
            self.ranges.append(ranges)
            if hi > lo:
                part = shard.shard_rows(t, mode, lo, hi)
                self.reps.append(build_hbcsf(part, allmode_order(t.dims, mode)))
                if part.nnz:
                    idx = torch.empty((part.nnz, t.order), dtype=torch.int32, device="cuda")
                    N.call("hbk_coo_export_device", part._dev().ptr, C.c_void_p(idx.data_ptr()), None,
                           None, N.stream_ptr())
                    for d in range(t.order):
                        if d != mode:
                            u = torch.unique(idx[:, d]).long()
                            refs[d].append(u)
                            self.needed_by[mode][d] = u
                    del idx
            else:
                self.reps.append(None)
        # rows of factor d this rank's MTTKRPs of the other modes read
        self.needed = [torch.unique(torch.cat(r)) if r else torch.zeros(0, dtype=torch.long, device="cuda")
                       for r in refs]

    def __call__(self, mode: int, factors32, skip_unowned: bool = False):
        from .kernels import mttkrp_device

        lo, hi = self.ranges[mode][self.me]
        rep = self.reps[mode]
        ref = factors32[(mode + 1) % len(factors32)]
        if rep is None:
            return ref.new_zeros((0, ref.shape[1]))
        fs = list(factors32)
        fs[mode] = factors32[mode][: hi - lo]  # shape only; factors[mode] is not read
        y, _ = mttkrp_device(rep, fs, mode, skip_unowned=skip_unowned)
        return y

    def owned_rows(self, mode: int, rank: int = 32):
        """This rank's output rows of ``mode`` that some bucket owns (local
        indices, device int32), or None."""
        from .kernels import plan_for

        rep = self.reps[mode]
        return None if rep is None else plan_for(rep, mode, rank).owned_rows()


class RowExchange:
    """Touched-rows exchange of one factor: after factor d is
    updated, each rank receives only the rows its own shards of the other
    modes read, from the ranks that own them — one all_to_all of row blocks
    instead of replicating the whole factor.  The send/receive index lists
    are agreed once (two small all_to_alls)."""

    def __init__(self, torch, dist, needed, ranges, me: int, group=None):
        world = len(ranges)
        self.group = group
        dev = needed.device
        parts, splits = [], []
        for r, (lo, hi) in enumerate(ranges):
            sel = needed[(needed >= lo) & (needed < hi)] if r != me else needed[:0]
            parts.append(sel)
            splits.append(int(sel.numel()))
        self.recv_idx = torch.cat(parts) if parts else needed[:0]
        self.recv_splits = splits
        cnt_out = torch.tensor(splits, dtype=torch.long, device=dev)
        cnt_in = torch.empty_like(cnt_out)
        dist.all_to_all_single(cnt_in, cnt_out, group=group)
        self.send_splits = [int(x) for x in cnt_in.tolist()]
        send_idx = torch.empty(sum(self.send_splits), dtype=torch.long, device=dev)
        dist.all_to_all_single(send_idx, self.recv_idx, output_split_sizes=self.send_splits,
                               input_split_sizes=self.recv_splits, group=group)
        self.send_idx = send_idx
        self.rows_in = int(self.recv_idx.numel())

    def __call__(self, torch, dist, F):
        self.finish(torch, self.start(torch, dist, F), F)

    def start(self, torch, dist, F):
        """Issue the exchange asynchronously; returns the pending handle."""
        width = F.shape[1]
        send = F.index_select(0, self.send_idx)
        recv = torch.empty((self.rows_in, width), dtype=F.dtype, device=F.device)
        work = dist.all_to_all_single(recv, send, output_split_sizes=self.recv_splits,
                                      input_split_sizes=self.send_splits, group=self.group,
                                      async_op=True)
        return work, recv, send

    def finish(self, torch, pending, F):
        """Wait for a started exchange (the current stream waits on it) and
        scatter the received rows into F."""
        work, recv, _ = pending
        work.wait()
        if self.rows_in:
            F.index_copy_(0, self.recv_idx, recv)


class SplitExchange:
    """Touched-rows exchange of factor d split by urgency: the rows the very
    next MTTKRP (mode d+1) reads are exchanged before it starts; the rows only
    later modes read are sent asynchronously and scattered at the next
    exchange call, so their transfer overlaps mode d+1's MTTKRP and row update
    (round-1 verdict: overlap the exchange with the next mode)."""

    def __init__(self, torch, dist, needed_by, d, ranges, me, group=None, device=None):
        order = len(needed_by)
        nxt = (d + 1) % order
        dev = device if device is not None else torch.device("cpu")
        empty = torch.zeros(0, dtype=torch.long, device=dev)

        def rows(m):
            x = needed_by[m][d]
            return empty if x is None else torch.as_tensor(x, dtype=torch.long).to(dev)

        crit = torch.unique(rows(nxt))
        later = [rows(m) for m in range(order) if m not in (d, nxt)]
        rest = torch.unique(torch.cat(later)) if later else empty
        if rest.numel() and crit.numel():
            rest = rest[~torch.isin(rest, crit)]
        self.crit = RowExchange(torch, dist, crit, ranges, me, group)
        self.rest = RowExchange(torch, dist, rest, ranges, me, group)
        self.rows_in = self.crit.rows_in + self.rest.rows_in


def cp_als_distributed(t: CooTensor, rank: int = 32, max_iters: int = 50, fit_tol: float = 1e-8,
                       seed: int = 0, *, group=None, local_mttkrp=None, ranges=None,
                       device=None, exchange: str = "touched", needed=None, needed_by=None,
                       sweep_hook=None):
    """CP-ALS over ``world`` processes, each owning a row range of every mode.

    Every rank passes the same tensor ``t`` (it is canonicalised and sharded
    locally).  Returns the same (KruskalModel, [AlsIteration]) as ``cp_als`` on
    every rank.  ``local_mttkrp(mode, factors32) -> (rows_g, R)`` and
    ``ranges`` (per mode, the row ranges of all ranks) replace the GPU shards
    (used by the CPU tests); by default the HB-CSF shards are built on the GPU
    and the collectives run on NCCL.  ``exchange``: "touched" (default)
    moves only the factor rows each rank's shards read — split by urgency when
    ``needed_by[mode][d]`` (the row ids of factor d this rank's shard of
    ``mode`` reads; derived from the GPU shards by default) is known: the rows
    the next mode reads go first, the rest overlap that mode's MTTKRP
    (``SplitExchange``); with only ``needed[d]`` (the union) one exchange per
    factor — and "full" replicates every updated factor.

    Factors are kept in fp32 (the MTTKRP's input precision) as raw matrices
    with per-column scales s_d: the true factor is F_d diag(s_d).  The scales
    absorb the column normalisation (cpd.py:187-195) and fold into the 32x32
    update matrix, so no pass over the factors is spent on it; Grams, fit
    terms and the pseudo-inverse stay fp64 (cpd.py:39-83,176-184)."""
    import torch

    dist = _dist()
    world = dist.get_world_size(group)
    me = dist.get_rank(group)
    if rank < 1:
        raise ValueError("rank must be at least 1")
    if max_iters < 0:
        raise ValueError("max_iters must be nonnegative")
    owned_rows = None
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
        owned_rows = lambda mode: shards.owned_rows(mode, rank)  # noqa: E731
        if needed is None and needed_by is None:
            needed_by = shards.needed_by
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
    if exchange not in ("touched", "full"):
        raise ValueError("exchange must be 'touched' or 'full'")
    own = [ranges[d][me] for d in range(order)]

    def allreduce_(x):
        dist.all_reduce(x, group=group)
        return x

    touched = split = None
    pending = {}  # factor d -> its deferred (SplitExchange.rest) exchange in flight
    if exchange == "touched" and world > 1 and needed_by is not None:
        split = [SplitExchange(torch, dist, needed_by, d, ranges[d], me, group, device)
                 for d in range(order)]
    elif exchange == "touched" and world > 1 and needed is not None:
        touched = [RowExchange(torch, dist, torch.as_tensor(needed[d], dtype=torch.long).to(device),
                               ranges[d], me, group) for d in range(order)]

    def drain(f32):
        for d in list(pending):
            split[d].rest.finish(torch, pending.pop(d), f32[d])

    def replicate(d, f32):
        """Replicate factor d's rows: rank r broadcasts its contiguous rows."""
        if world == 1:
            return
        for r, (lo, hi) in enumerate(ranges[d]):
            if hi > lo:
                # ranges are indexed by group rank; broadcast wants the global rank
                src = dist.get_global_rank(group, r) if group is not None else r
                dist.broadcast(f32[d][lo:hi], src=src, group=group)

    def exchange_rows(d, f32):
        if split is not None:
            drain(f32)  # the previous factor's deferred rows (overlapped this mode's MTTKRP)
            split[d].crit(torch, dist, f32[d])
            pending[d] = split[d].rest.start(torch, dist, f32[d])
        elif touched is not None:
            touched[d](torch, dist, f32[d])
        else:
            replicate(d, f32)

    def finalize(f32):
        if split is not None:
            drain(f32)
        if touched is not None or split is not None:  # the model needs every row of every factor
            for d in range(order):
                replicate(d, f32)

    return als_fp32(torch, dims=dims, rank=rank, max_iters=max_iters, fit_tol=fit_tol, seed=seed,
                    device=device, own=own, local_mttkrp=local_mttkrp,
                    norm_x=_value_norm(torch, t), allreduce_=allreduce_,
                    exchange_rows=exchange_rows, finalize=finalize, sweep_hook=sweep_hook,
                    owned_rows=owned_rows)


def als_fp32(torch, *, dims, rank, max_iters, fit_tol, seed, device, own, local_mttkrp, norm_x,
             allreduce_=lambda x: x, exchange_rows=lambda d, f32: None, finalize=lambda f32: None,
             sweep_hook=None, owned_rows=None):
    """The CP-ALS sweep loop (cpd.py:198-271) on fp32 factors with folded
    column scales, for a rank owning rows ``own[d]`` of every factor.
    ``local_mttkrp(mode, f32)`` returns this rank's (rows, R) MTTKRP (or a
    (rows, OpCount) pair); the hooks do the collectives (identity on one
    process).  Used by cp_als_distributed and by cp_als at R = 32."""
    order = len(dims)
    import os

    fused = device.type == "cuda" and rank == 32 and os.environ.get("HBK_ALS_FUSED", "1") != "0"
    rng = np.random.default_rng(seed)
    f32 = [torch.from_numpy(rng.random((dim, rank))).to(device=device, dtype=torch.float32)
           for dim in dims]  # cpd.py:231-232, identical on every rank
    scales = [np.ones(rank) for _ in dims]

    def mttkrp(mode, skip_unowned=False):
        # skip_unowned (with owned_rows): rows no bucket owns are not written —
        # the row update then reads only the owned rows
        skip_unowned = skip_unowned and os.environ.get("HBK_SKIP_UNOWNED", "1") != "0"
        r = local_mttkrp(mode, f32, skip_unowned=True) if skip_unowned else local_mttkrp(mode, f32)
        return r if isinstance(r, tuple) else (r, None)

    def gram_raw(local):
        g = torch.zeros((rank, rank), dtype=torch.float64, device=device)
        for a in range(0, local.shape[0], 1 << 20):  # fp32 partials over <= 1M rows
            c = local[a: a + (1 << 20)]
            g += (c.T @ c).double()
        return g

    def true_gram(d, g_raw):
        s = scales[d]
        g = (g_raw.cpu().numpy() * np.outer(s, s))
        return (g + g.T) * 0.5

    def sync():
        if device.type == "cuda":
            torch.cuda.synchronize(device)

    grams = []
    for d in range(order):
        lo, hi = own[d]
        grams.append(true_gram(d, allreduce_(gram_raw(f32[d][lo:hi]))))
    last = order - 1

    def fit_value(inner):
        norm_hat_sq = float((hadamard_all_but(grams, last) * grams[last]).sum())
        err_sq = max(norm_x * norm_x + norm_hat_sq - 2.0 * inner, 0.0)
        return 1.0 - math.sqrt(err_sq) / norm_x

    def colscale(mode):
        c = np.ones(rank)
        for d in range(order):
            if d != mode:
                c = c * scales[d]
        return c

    y0 = mttkrp(last)[0].double()
    lo, hi = own[last]
    inner0 = float((y0 * torch.from_numpy(colscale(last)).to(device)
                    * (f32[last][lo:hi].double() * torch.from_numpy(scales[last]).to(device))).sum())
    history = [AlsIteration(0, fit_value(float(allreduce_(torch.tensor([inner0], dtype=torch.float64,
                                                                      device=device)).item())),
                            0.0, (), ())]
    del y0
    lam = None
    inner_t = torch.zeros(1, dtype=torch.float64, device=device)
    # CUDA + fused: the sweep is pipelined — mode n+1's MTTKRP (which needs
    # only the factors) is queued right behind mode n's row update, and the
    # host reads mode n's Gram and forms M_{n+1} = pinv(V) while that MTTKRP
    # runs, so the GPU does not idle on host round trips.  mode_seconds are
    # then device times (CUDA events, MTTKRP start -> update end).
    pipelined = fused
    if pipelined:
        m_pin = torch.empty((rank, rank), dtype=torch.float32, pin_memory=True)
        w_pin = torch.empty(rank, dtype=torch.float32, pin_memory=True)
        g_pin = torch.empty((rank, rank), dtype=torch.float64, pin_memory=True)
        m_dev = torch.empty((rank, rank), dtype=torch.float32, device=device)
        w_dev = torch.empty(rank, dtype=torch.float32, device=device)
        ev_g = torch.cuda.Event()
        in_pin = torch.empty(1, dtype=torch.float64, pin_memory=True)
    ahead = None

    def update(mode, y, with_inner, use_list=False):
        """F_mode <- Y M (rows this rank owns), the raw Gram of the new rows;
        the fit term into inner_t when with_inner.  use_list: only the rows
        some bucket owns (owned_rows(mode)); the others are zero in Y and
        have been zero in F since the first sweep wrote them."""
        c = colscale(mode)
        # F_true = (Y_raw diag(c)) V^+  ->  M = diag(c) V^+, new scales 1
        m64 = c[:, None] * pinv_spsd(hadamard_all_but(grams, mode))
        lo, hi = own[mode]
        dst = f32[mode][lo:hi]
        g_raw = torch.zeros((rank, rank), dtype=torch.float64, device=device)
        if fused:
            from . import _native as N
            import ctypes as C

            if pipelined:  # page-locked staging, no host-side wait on the stream
                m_pin.copy_(torch.from_numpy(m64))
                w_pin.copy_(torch.from_numpy(c))
                m_dev.copy_(m_pin, non_blocking=True)
                w_dev.copy_(w_pin, non_blocking=True)
                m32, w32 = m_dev, w_dev
            else:
                m32 = torch.from_numpy(m64).to(device=device, dtype=torch.float32).contiguous()
                w32 = torch.from_numpy(c).to(device=device, dtype=torch.float32)
            rows_l = owned_rows(mode) if (use_list and owned_rows is not None) else None
            # (the MTTKRP of such a sweep leaves unowned rows of Y unwritten)
            if rows_l is not None and hi > lo:
                N.call("hbk_als_update_rows", C.c_void_p(y.data_ptr()),
                       C.c_void_p(rows_l.data_ptr()), int(rows_l.numel()), int(rank),
                       C.c_void_p(m32.data_ptr()), C.c_void_p(w32.data_ptr()),
                       C.c_void_p(dst.data_ptr()), C.c_void_p(g_raw.data_ptr()),
                       C.c_void_p(inner_t.data_ptr()) if with_inner else None, N.stream_ptr())
            elif hi > lo:
                N.call("hbk_als_update", C.c_void_p(y.data_ptr()), int(hi - lo), int(rank),
                       C.c_void_p(m32.data_ptr()), C.c_void_p(w32.data_ptr()),
                       C.c_void_p(dst.data_ptr()), C.c_void_p(g_raw.data_ptr()),
                       C.c_void_p(inner_t.data_ptr()) if with_inner else None, N.stream_ptr())
            elif with_inner:
                inner_t.zero_()
            return g_raw, (inner_t.clone() if with_inner else None)
        fm = y @ torch.from_numpy(m64).to(device=device, dtype=torch.float32)
        dst.copy_(fm)
        g_raw = gram_raw(dst)
        inner_m = None
        if with_inner:  # sum_r c_r <Y[:, r], F[:, r]>, fp32 chunks, fp64 total
            cw = torch.from_numpy(c).to(device=device, dtype=fm.dtype)
            inner_m = torch.zeros(1, dtype=torch.float64, device=device)
            for a in range(0, fm.shape[0], 1 << 20):
                inner_m += ((y[a: a + (1 << 20)] * fm[a: a + (1 << 20)]).sum(0).double()
                            * cw.double()).sum()
        return g_raw, inner_m

    def set_gram(mode, g, it):
        if not np.isfinite(g).all():
            raise NumericalError(f"non-finite factor for mode {mode} in ALS sweep {it}", iteration=it)
        scales[mode] = np.ones(rank)
        grams[mode] = (g + g.T) * 0.5

    for it in range(1, max_iters + 1):
        seconds, ops = [], []
        inner = 0.0
        sweep_tic = time.perf_counter()
        if pipelined:
            # mode_seconds[n]: from mode n's MTTKRP launch to mode n+1's (its
            # update, Gram read-back and row exchange included); the last mode
            # runs to the end of the sweep's exchange
            evs = [torch.cuda.Event(enable_timing=True) for _ in range(order + 1)]
            # from the second sweep on the row update reads only owned rows
            lists = owned_rows is not None and it > 1
            if ahead is not None:  # mode 0 was launched during the previous sweep's fit
                evs[0], pending = ahead
                ahead = None
            else:
                evs[0].record()
                pending = mttkrp(0, lists)
            for mode in range(order):
                y, op = pending
                y = y.float().contiguous()
                ops.append(op)
                g_raw, inner_m = update(mode, y, mode == last, use_list=lists)
                if inner_m is not None:
                    inner = inner_m
                g_pin.copy_(allreduce_(g_raw), non_blocking=True)
                ev_g.record()
                exchange_rows(mode, f32)
                if mode == last:
                    in_pin.copy_(allreduce_(inner.reshape(1)), non_blocking=True)
                evs[mode + 1].record()
                if mode + 1 < order:
                    pending = mttkrp(mode + 1, lists)
                elif it < max_iters:
                    # the next sweep's first MTTKRP needs only the factors:
                    # queue it now, so it runs while the host computes the fit
                    # (if the fit converges, its output is simply dropped)
                    ev0 = torch.cuda.Event(enable_timing=True)
                    ev0.record()
                    ahead = (ev0, mttkrp(0, owned_rows is not None))
                ev_g.synchronize()
                set_gram(mode, g_pin.numpy().copy(), it)
                del y
            evs[order].synchronize()
            seconds = [evs[m].elapsed_time(evs[m + 1]) * 1e-3 for m in range(order)]
            inner_val = float(in_pin[0])
        else:
            for mode in range(order):
                sync()
                tic = time.perf_counter()
                y, op = mttkrp(mode)
                y = y.float().contiguous()
                ops.append(op)
                g_raw, inner_m = update(mode, y, mode == last)
                if inner_m is not None:
                    inner = inner_m
                set_gram(mode, allreduce_(g_raw).cpu().numpy(), it)
                exchange_rows(mode, f32)
                del y
                sync()
                seconds.append(time.perf_counter() - tic)
            if not torch.is_tensor(inner):
                inner = torch.zeros(1, dtype=torch.float64, device=device)
            inner_val = float(allreduce_(inner.reshape(1)).item())
        new_fit = fit_value(inner_val)
        lam = _normalize_scales(scales, grams)
        if not math.isfinite(new_fit):
            raise NumericalError(f"non-finite fit in ALS sweep {it}", iteration=it)
        if sweep_hook is not None:  # host wall clock of the whole sweep
            sweep_hook(it, time.perf_counter() - sweep_tic)
        delta = new_fit - history[-1].fit
        history.append(AlsIteration(it, new_fit, delta, tuple(seconds),
                                    tuple(ops) if all(o is not None for o in ops) else ()))
        if abs(delta) < fit_tol:
            break
    if len(history) == 1:
        lam = _normalize_scales(scales, grams)
    finalize(f32)
    full = [(f32[d].double() * torch.from_numpy(scales[d]).to(device)).cpu().numpy()
            for d in range(order)]
    return KruskalModel(lam=lam, factors=tuple(full)), history


def _normalize_scales(scales, grams):
    """Column normalisation (cpd.py:187-195) applied to the scale vectors:
    norms from diag of the true Grams; F_d diag(s_d) -> F_d diag(s_d / n_d)."""
    lam = None
    for d in range(len(scales)):
        n = np.sqrt(np.maximum(np.diag(grams[d]), 0.0))
        n = np.where(n > 0.0, n, 1.0)
        scales[d] = scales[d] / n
        grams[d] = grams[d] / np.outer(n, n)
        lam = n.copy() if lam is None else lam * n
    return lam


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
