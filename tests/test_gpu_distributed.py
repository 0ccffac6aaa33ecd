"""GPU checks of the row-sharded path: rebased shards reproduce the full
MTTKRP row for row, and cp_als_distributed on a one-rank NCCL group matches
the single-GPU cp_als (the multi-rank collectives are covered on CPU with
gloo in test_distributed_cpu.py)."""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest

from oracle import tenkit_port as P

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def hb():
    import paper_1904_03329_b200 as hb

    return hb


def _powerlaw(rng, dims, nnz):
    cols = [np.minimum(np.floor(np.exp(rng.random(nnz) * np.log(d + 1))) - 1, d - 1) for d in dims]
    idx = np.stack(cols, 1).astype(np.uint32)
    return P.canonical(idx, rng.random(nnz) + 0.01)


@pytest.mark.parametrize("world", [2, 3, 8])
def test_shards_concatenate_to_full_mttkrp(hb, world):
    from paper_1904_03329_b200 import shard

    rng = np.random.default_rng(11 + world)
    dims = (120, 90, 300)
    idx, vals = _powerlaw(rng, dims, 20000)
    t = hb.CooTensor(dims, idx, vals, sorted_under=(0, 1, 2))
    fs = [rng.random((d, 32)).astype(np.float32).astype(np.float64) for d in dims]
    for mode in range(3):
        mo = hb.allmode_order(dims, mode)
        ref, _ = P.mttkrp_hbcsf(P.hbcsf(idx, vals, dims, mo), fs, mode)
        hist = shard.slice_histogram(t, mode).cpu().numpy()
        assert np.array_equal(hist, np.bincount(idx[:, mode], minlength=dims[mode]))
        ranges = shard.plan_row_ranges(hist, world)
        parts = []
        for lo, hi in ranges:
            if hi == lo:
                continue
            part = shard.shard_rows(t, mode, lo, hi)
            assert part.dims[mode] == hi - lo
            h = hb.split_fibers(hb.build_hbcsf(part, mo), hb.SplitConfig())
            f = list(fs)
            f[mode] = np.zeros((hi - lo, 32))
            y, _ = hb.mttkrp_hbcsf(h, f, mode)
            parts.append(y)
        y = np.concatenate(parts)
        assert y.shape == ref.shape
        assert P.row_deviation(y, ref) <= 1e-4


def test_cp_als_distributed_single_rank_matches_cp_als(hb):
    import torch
    import torch.distributed as dist

    from paper_1904_03329_b200.distributed import cp_als_distributed

    rng = np.random.default_rng(5)
    dims = (40, 30, 50)
    idx, vals = _powerlaw(rng, dims, 6000)
    t = hb.CooTensor(dims, idx, vals, sorted_under=(0, 1, 2))
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        m1, h1 = cp_als_distributed(t, rank=8, max_iters=5, fit_tol=1e-14, seed=3)
    finally:
        dist.destroy_process_group()
    m0, h0 = hb.cp_als(t, rank=8, max_iters=5, fit_tol=1e-14, seed=3)
    assert len(h0) == len(h1)
    assert np.allclose([h.fit for h in h1], [h.fit for h in h0], atol=1e-5, rtol=0)
    assert np.allclose(m1.lam, m0.lam, rtol=1e-3)
    fits_ref, _, _ = P.cp_als(idx, vals, dims, rank=8, max_iters=5, fit_tol=1e-14, seed=3)
    assert np.allclose([h.fit for h in h1], fits_ref, atol=1e-5, rtol=0)


@pytest.mark.parametrize("kernel", ["mma", "tc"])
@pytest.mark.parametrize("rows", [1, 255, 1000, 70000])
def test_als_update_kernel_matches_fp64(rows, kernel, monkeypatch):
    """hbk_als_update: F = Y M, Gram = F^T F, weighted <Y, F> against an fp64
    torch restatement (fp32 kernel arithmetic, so 1e-5 relative) — the
    default mma.sync kernel and the tcgen05 one (HBK_ALS_KERNEL=tc)."""
    import ctypes as C

    monkeypatch.setenv("HBK_ALS_KERNEL", kernel)

    import torch

    from paper_1904_03329_b200 import _native as N

    g = torch.Generator(device="cuda").manual_seed(rows)
    Y = torch.rand((rows, 32), device="cuda", generator=g) - 0.3
    M = torch.rand((32, 32), device="cuda", generator=g) - 0.5
    w = torch.rand(32, device="cuda", generator=g) + 0.5
    F = torch.empty_like(Y)
    gram = torch.empty((32, 32), dtype=torch.float64, device="cuda")
    inner = torch.empty(1, dtype=torch.float64, device="cuda")
    N.call("hbk_als_update", C.c_void_p(Y.data_ptr()), rows, 32, C.c_void_p(M.data_ptr()),
           C.c_void_p(w.data_ptr()), C.c_void_p(F.data_ptr()), C.c_void_p(gram.data_ptr()),
           C.c_void_p(inner.data_ptr()), N.stream_ptr())
    F64 = Y.double() @ M.double()
    assert torch.allclose(F.double(), F64, rtol=1e-5, atol=1e-5)
    G64 = F64.T @ F64
    assert torch.allclose(gram, G64, rtol=1e-5, atol=1e-4 * float(G64.abs().max()) * 1e-2 + 1e-6)
    I64 = float(((Y.double() * w.double()) * F64).sum())
    assert abs(float(inner) - I64) <= 1e-5 * max(1.0, abs(I64))
    with pytest.raises(ValueError):
        N.call("hbk_als_update", C.c_void_p(Y.data_ptr()), rows, 16, C.c_void_p(M.data_ptr()),
               None, C.c_void_p(F.data_ptr()), C.c_void_p(gram.data_ptr()), None, N.stream_ptr())


@pytest.mark.parametrize("kernel", ["mma", "tc"])
@pytest.mark.parametrize("rows", [1, 37, 5000, 70001])
def test_als_update_rows_matches_full_update(rows, kernel, monkeypatch):
    """hbk_als_update_rows over the nonzero rows of Y equals hbk_als_update
    over all rows when the other rows are zero (F, Gram, fit term); rows not
    listed keep their previous F contents."""
    import ctypes as C

    monkeypatch.setenv("HBK_ALS_KERNEL", kernel)

    import torch

    from paper_1904_03329_b200 import _native as N

    g = torch.Generator(device="cuda").manual_seed(rows + 1)
    Y = torch.rand((rows, 32), device="cuda", generator=g) - 0.3
    keep = torch.rand(rows, device="cuda", generator=g) < 0.6
    keep[0] = True
    Y[~keep] = 0.0
    lst = torch.nonzero(keep).flatten().to(torch.int32)
    M = torch.rand((32, 32), device="cuda", generator=g) - 0.5
    w = torch.rand(32, device="cuda", generator=g) + 0.5
    outs = []
    for use_list in (False, True):
        F = torch.full_like(Y, 7.0)
        gram = torch.empty((32, 32), dtype=torch.float64, device="cuda")
        inner = torch.empty(1, dtype=torch.float64, device="cuda")
        if use_list:
            N.call("hbk_als_update_rows", C.c_void_p(Y.data_ptr()), C.c_void_p(lst.data_ptr()),
                   int(lst.numel()), 32, C.c_void_p(M.data_ptr()), C.c_void_p(w.data_ptr()),
                   C.c_void_p(F.data_ptr()), C.c_void_p(gram.data_ptr()),
                   C.c_void_p(inner.data_ptr()), N.stream_ptr())
        else:
            N.call("hbk_als_update", C.c_void_p(Y.data_ptr()), rows, 32, C.c_void_p(M.data_ptr()),
                   C.c_void_p(w.data_ptr()), C.c_void_p(F.data_ptr()), C.c_void_p(gram.data_ptr()),
                   C.c_void_p(inner.data_ptr()), N.stream_ptr())
        outs.append((F, gram, inner))
    (F0, g0, i0), (F1, g1, i1) = outs
    assert torch.equal(F1[keep], F0[keep])  # same MMA arithmetic per row
    assert bool((F1[~keep] == 7.0).all())   # unlisted rows untouched
    # the listed rows form different 16-row MMA subtiles: the Gram and the fit
    # term agree to fp32 accumulation order
    assert torch.allclose(g1, g0, rtol=1e-6, atol=1e-6 * float(g0.abs().max()))
    assert abs(float(i1) - float(i0)) <= 1e-6 * max(1.0, abs(float(i0)))
    assert torch.equal(g1, g1.T)
