"""Multi-process (gloo, world size 2) tests of the row-sharded CP-ALS and the
factor exchange — the host logic of the NCCL path, run on CPU.

Each rank's local MTTKRP is the oracle over its rebased row shard (the GPU
kernels are covered by the -m gpu tests); the collectives, padding, ALS
algebra, fit and normalisation are the product code
(paper_1904_03329_b200.distributed)."""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import tenkit_port as P


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _tensor(seed=3, dims=(23, 17, 29), nnz=900):
    rng = np.random.default_rng(seed)
    idx = np.stack([rng.integers(0, d, nnz) for d in dims], 1).astype(np.uint32)
    # a few heavy rows so the nnz-balanced ranges are uneven
    idx[: nnz // 4, 0] = 0
    vals = rng.random(nnz) + 0.05
    return P.canonical(idx, vals)


def _worker(rank, world, port, q, job):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q.put((rank, job(rank, world)))
    except Exception as e:  # surface the failure in the parent
        q.put((rank, e))
    finally:
        dist.destroy_process_group()


def _run(job, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, job)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    for r, v in out.items():
        if isinstance(v, Exception):
            raise v
    return [out[r] for r in range(world)]


# --------------------------------------------------------------- jobs (picklable)
def _job_allgather(rank, world):
    from paper_1904_03329_b200.distributed import allgather_rows

    full = torch.arange(6 * 3, dtype=torch.float64).reshape(6, 3)
    ok = True
    # uneven ranges, and a rank with an empty range
    for ranges in ([(0, 5), (5, 6)], [(0, 6), (6, 6)], [(0, 0), (0, 6)]):
        ranges = ranges if world == 2 else [(0, 6)]
        lo, hi = ranges[rank]
        got = allgather_rows(torch, dist, full[lo:hi].clone(), ranges)
        ok = ok and bool(torch.equal(got, full))
    return ok


def _local_mttkrp_factory(idx, vals, dims, ranges, rank):
    def local(mode, factors32):
        lo, hi = ranges[mode][rank]
        keep = (idx[:, mode] >= lo) & (idx[:, mode] < hi)
        sidx = idx[keep].copy()
        sidx[:, mode] -= lo
        sdims = list(dims)
        sdims[mode] = hi - lo
        fs = [f.double().numpy() for f in factors32]
        fs[mode] = np.zeros((hi - lo, fs[(mode + 1) % len(fs)].shape[1]))
        mo = P.allmode_order(dims, mode)
        h = P.hbcsf(sidx, vals[keep], tuple(sdims), mo)
        y, _ = P.mttkrp_hbcsf(h, fs, mode)
        return torch.from_numpy(y)
    return local


def _needed_rows(idx, dims, ranges, rank):
    """Rows of factor d read by this rank's shards of the other modes."""
    need = []
    for d in range(3):
        rows = set()
        for n in range(3):
            if n == d:
                continue
            lo, hi = ranges[n][rank]
            keep = (idx[:, n] >= lo) & (idx[:, n] < hi)
            rows.update(idx[keep, d].tolist())
        need.append(np.array(sorted(rows), dtype=np.int64))
    return need


def _needed_by(idx, dims, ranges, rank):
    """Rows of factor d read by this rank's shard of each mode."""
    out = [[None] * 3 for _ in range(3)]
    for n in range(3):
        lo, hi = ranges[n][rank]
        keep = (idx[:, n] >= lo) & (idx[:, n] < hi)
        for d in range(3):
            if d != n:
                out[n][d] = np.unique(idx[keep, d]).astype(np.int64)
    return out


def _job_cpd(rank, world, exchange="full", group=None):
    from paper_1904_03329_b200.coo import CooTensor
    from paper_1904_03329_b200.distributed import cp_als_distributed
    from paper_1904_03329_b200.shard import plan_row_ranges

    idx, vals = _tensor()
    dims = (23, 17, 29)
    t = CooTensor(dims, idx, vals, sorted_under=(0, 1, 2))
    ranges = [plan_row_ranges(np.bincount(idx[:, m], minlength=dims[m]), world) for m in range(3)]
    local = _local_mttkrp_factory(idx, vals, dims, ranges, rank)
    needed = _needed_rows(idx, dims, ranges, rank) if exchange == "touched" else None
    needed_by = None
    if exchange == "split":
        exchange, needed_by = "touched", _needed_by(idx, dims, ranges, rank)
    model, hist = cp_als_distributed(t, rank=4, max_iters=6, fit_tol=1e-14, seed=7,
                                     local_mttkrp=local, ranges=ranges, exchange=exchange,
                                     needed=needed, needed_by=needed_by, group=group)
    return [h.fit for h in hist], model.lam, [f for f in model.factors], ranges


def _job_cpd_touched(rank, world):
    return _job_cpd(rank, world, exchange="touched")


def _job_cpd_split(rank, world):
    return _job_cpd(rank, world, exchange="split")


def _job_cpd_subgroup(rank, world):
    """Global ranks 1..2 of a world-3 job decompose in a subgroup (group
    ranks 0..1); global rank 0 stays out."""
    sub = dist.new_group([1, 2])
    if rank == 0:
        return None
    res = {}
    for ex in ("full", "touched", "split"):
        res[ex] = _job_cpd(dist.get_rank(sub), 2, exchange=ex, group=sub)
    return res


def test_allgather_rows_uneven_world2():
    assert _run(_job_allgather) == [True, True]


def test_cp_als_distributed_matches_single_process_oracle():
    res = _run(_job_cpd)
    (fits0, lam0, f0, ranges), (fits1, lam1, f1, _) = res
    # the nnz-balanced ranges are uneven (the heavy row 0 of mode 0)
    assert ranges[0][0] != (0, 23 // 2)
    # every rank returns the same model
    assert fits0 == fits1
    assert np.array_equal(lam0, lam1)
    for a, b in zip(f0, f1):
        assert np.array_equal(a, b)
    idx, vals = _tensor()
    fits_ref, _, lam_ref = P.cp_als(idx, vals, (23, 17, 29), rank=4, max_iters=6, fit_tol=1e-14,
                                    seed=7)
    # fp32 factor copies feed the MTTKRP (as on the GPU); the fits agree to
    # fp32 rounding of the factors
    assert len(fits0) == len(fits_ref)
    assert np.allclose(fits0, fits_ref, atol=2e-6, rtol=0)
    assert np.allclose(lam0, lam_ref, rtol=2e-4)


@pytest.mark.parametrize("world", [2, 3])
def test_touched_rows_exchange_matches_full_replication(world):
    """Touched-rows exchange (each rank receives only the factor rows its
    shards read) — in one piece, and split into the rows the next mode reads
    plus a deferred remainder overlapping that mode (SplitExchange) — gives
    the same model as full replication, on every rank."""
    full = _run(_job_cpd, world)
    for job in (_job_cpd_touched, _job_cpd_split):
        touched = _run(job, world)
        for r in range(world):
            assert np.allclose(touched[r][0], full[0][0], atol=1e-12, rtol=0)
            assert np.allclose(touched[r][1], full[0][1], rtol=1e-12)
            for a, b in zip(touched[r][2], full[0][2]):
                assert np.allclose(a, b, rtol=1e-10, atol=1e-12)


def test_cp_als_distributed_in_a_subgroup():
    """with a non-default group the row owners are group ranks;
    the broadcasts must address them by global rank.  A subgroup {1, 2} of
    a world-3 job reproduces the world-2 default-group model."""
    ref = _run(_job_cpd, 2)
    sub = _run(_job_cpd_subgroup, 3)
    assert sub[0] is None
    for r in (1, 2):
        for ex in ("full", "touched", "split"):
            fits, lam, fac, _ = sub[r][ex]
            assert np.allclose(fits, ref[0][0], atol=1e-12, rtol=0)
            assert np.allclose(lam, ref[0][1], rtol=1e-12)
            for a, b in zip(fac, ref[0][2]):
                assert np.allclose(a, b, rtol=1e-10, atol=1e-12)
