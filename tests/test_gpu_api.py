"""GPU tests of the drop-in API beyond the golden fixtures: the reference's
hand examples and argument guards (test_kernels.py:38-56, 274-308), edge
cases (empty, single nonzero, order 4, ranks the fast path does not take),
device-tensor inputs, and parity against the CPU oracle on power-law tensors
large enough to exercise heavy-slice chunking and all three buckets."""
from __future__ import annotations

import numpy as np
import pytest

from helpers import row_dev
from oracle import loops
from oracle import tenkit_port as P

pytestmark = pytest.mark.gpu

TOL = 1e-4


@pytest.fixture(scope="module")
def hb():
    import paper_1904_03329_b200 as hb

    return hb


def _rand(rng, dims, nnz):
    cap = int(np.prod(dims))
    flats = rng.choice(cap, size=nnz, replace=False)
    idx = np.empty((nnz, len(dims)), dtype=np.int64)
    rem = flats
    for d in range(len(dims) - 1, -1, -1):
        idx[:, d] = rem % dims[d]
        rem //= dims[d]
    return idx.astype(np.uint32), rng.uniform(0.1, 1.0, nnz)


def _powerlaw(rng, dims, nnz, alpha=1.0):
    cols = []
    for d in dims:
        u = rng.random(nnz)
        x = np.exp(u * np.log(d + 1.0)) if alpha == 1.0 else 1.0 + u * d
        cols.append(np.minimum(np.floor(x).astype(np.int64) - 1, d - 1))
    idx = np.stack(cols, 1).astype(np.uint32)
    return P.canonical(idx, rng.uniform(0.1, 1.0, nnz))


# reference hand examples -------------------------------------------------
def test_coo_single_nonzero_hand_example(hb):
    t = hb.CooTensor((1, 1, 1), np.zeros((1, 3), dtype=np.int64), [5.0])
    f = [np.array([[0.0]]), np.array([[3.0]]), np.array([[7.0]])]
    out, ops = hb.mttkrp_coo(hb.canonicalize(t), f, 0)
    assert out[0, 0] == 105.0 and ops.total == 3


def test_csl_two_entry_hand_example(hb):
    t = hb.canonicalize(hb.CooTensor((1, 2, 2), np.array([[0, 0, 0], [0, 1, 1]]), [2.0, 3.0]))
    h = hb.build_hbcsf(t, (0, 1, 2))
    assert h.coo_part.nnz == 0 and h.csf_part.num_slices == 0
    assert len(h.csl_part.slice_idx) == 1
    f = [np.zeros((1, 1)), np.array([[1.0], [10.0]]), np.array([[1.0], [100.0]])]
    out, ops = hb.mttkrp_csl(h.csl_part, f, 0)
    assert out[0, 0] == 3002.0 and ops.total == 6


# edge cases --------------------------------------------------------------
def test_empty_tensor(hb):
    t = hb.canonicalize(hb.CooTensor((2, 3, 4), np.empty((0, 3), dtype=np.int64), np.empty(0)))
    assert t.nnz == 0 and t.sorted_under == (0, 1, 2)
    c = hb.build_csf(t, (0, 1, 2))
    assert all(p.tolist() == [0] for p in c.ptrs) and c.num_slices == 0
    h = hb.build_hbcsf(t, (0, 1, 2))
    assert h.nnz == 0
    f = [np.ones((d, 3)) for d in (2, 3, 4)]
    for rep in (t, c, h):
        y, ops = hb.mttkrp(rep, f, 0)
        assert y.shape == (2, 3) and not y.any() and ops.total == 0
    assert hb.split_fibers(c, hb.SplitConfig()) is c
    s = hb.assign_slice_blocks(c, hb.SplitConfig())
    assert s.num_blocks == 0 and len(s.multiplicities) == 0


def test_rows_without_nonzeros_are_zero(hb):
    idx = np.array([[3, 0, 1], [3, 1, 1], [7, 2, 0]], dtype=np.uint32)
    t = hb.CooTensor((10, 3, 2), idx, [1.0, 2.0, 3.0])
    f = [np.ones((10, 32)), np.ones((3, 32)), np.ones((2, 32))]
    y, _ = hb.mttkrp_hbcsf(hb.build_hbcsf(t, (0, 1, 2)), f, 0)
    assert np.allclose(y[3], 3.0) and np.allclose(y[7], 3.0)
    assert not np.delete(y, [3, 7], axis=0).any()


@pytest.mark.parametrize("rank", [1, 2, 4, 7, 12, 16, 32, 33, 48, 64, 96])
def test_ranks_match_loop_oracle(hb, rng, rank):
    idx, vals = _rand(rng, (9, 8, 7), 150)
    t = hb.CooTensor((9, 8, 7), idx, vals)
    f = [rng.standard_normal((d, rank)) for d in (9, 8, 7)]
    f = [x.astype(np.float32).astype(np.float64) for x in f]
    for mode in range(3):
        ref = loops.mttkrp_entries(idx, vals, (9, 8, 7), f, mode)
        h = hb.build_hbcsf(t, hb.allmode_order(t.dims, mode))
        for rep in (h, hb.split_fibers(h, hb.SplitConfig(2, 4, 2)), t):
            y, _ = hb.mttkrp(rep, f, mode)
            assert row_dev(y, ref) <= TOL


def test_fp64_mode_matches_loop_oracle(hb, rng):
    idx, vals = _rand(rng, (20, 15, 12), 900)
    t = hb.CooTensor((20, 15, 12), idx, vals)
    f = [rng.standard_normal((d, 32)) for d in (20, 15, 12)]
    for mode in range(3):
        ref = loops.mttkrp_entries(idx, vals, (20, 15, 12), f, mode)
        mo = hb.allmode_order(t.dims, mode)
        h = hb.split_fibers(hb.build_hbcsf(t, mo), hb.SplitConfig(3, 8, 2))
        for y, _ in (hb.mttkrp(h, f, mode, precision="fp64"), hb.mttkrp(t, f, mode, precision="fp64"),
                     hb.mttkrp(hb.build_csf(t, mo), f, mode, precision="fp64")):
            assert row_dev(y, ref) <= 1e-12
    with pytest.raises(ValueError):
        hb.mttkrp(h, f, 0, precision="fp16")


def test_order4_and_order5(hb, rng):
    for dims, nnz in (((6, 5, 4, 3), 200), ((4, 3, 5, 3, 2), 150)):
        idx, vals = _rand(rng, dims, nnz)
        t = hb.CooTensor(dims, idx, vals)
        f = [rng.random((d, 32)).astype(np.float32).astype(np.float64) for d in dims]
        for mode in range(len(dims)):
            ref = loops.mttkrp_entries(idx, vals, dims, f, mode)
            mo = hb.allmode_order(dims, mode)
            h = hb.build_hbcsf(t, mo)
            cfg = hb.SplitConfig(2, 4, 2)
            hs = hb.split_fibers(h, cfg)
            sched = hb.assign_slice_blocks(hs.csf_part, cfg)
            for y, ops in (hb.mttkrp(h, f, mode), hb.mttkrp_hbcsf(hs, f, mode, schedule=sched),
                           hb.mttkrp(hb.build_csf(t, mo), f, mode)):
                assert row_dev(y, ref) <= TOL
            # OpCount of the scheduled CSF path matches the oracle's executed-site count
            ref_h = P.split_hbcsf(P.hbcsf(idx, vals, dims, mo), 2)
            units, _ = P.block_schedule(ref_h["csf"], 4)
            _, k = P.mttkrp_hbcsf(ref_h, f, mode, units=units)
            _, ops = hb.mttkrp_hbcsf(hs, f, mode, schedule=sched)
            assert (ops.muls, ops.adds) == k


# argument guards (same exception types as the reference) -----------------
def test_argument_guards(hb, rng):
    idx, vals = _rand(rng, (5, 4, 3), 20)
    t = hb.CooTensor((5, 4, 3), idx, vals)
    h = hb.build_hbcsf(t, (0, 2, 1))
    f = [np.ones((5, 2)), np.ones((4, 2)), np.ones((3, 2))]
    with pytest.raises(ValueError):
        hb.mttkrp_hbcsf(h, f, 1)  # built for mode 0
    with pytest.raises(ValueError):
        hb.mttkrp_csf(h.csf_part, f, 2)
    with pytest.raises(ValueError):
        hb.mttkrp(h, f[:2], 0)
    with pytest.raises(ValueError):
        hb.mttkrp(h, [f[0], np.ones((4, 3)), f[2]], 0)
    with pytest.raises(ValueError):
        hb.mttkrp(h, [f[0], np.ones((5, 2)), f[2]], 0)
    with pytest.raises(ValueError):
        hb.mttkrp(h, [f[0], np.full((4, 2), np.inf), f[2]], 0)
    with pytest.raises(TypeError):
        hb.mttkrp(h.csf_part, f, 0, threads=2)  # mttkrp_csf takes no threads
    with pytest.raises(TypeError):
        hb.mttkrp([1, 2], f, 0)
    with pytest.raises(ValueError):
        hb.build_hbcsf(t, (0, 0, 1))
    # factors[mode] is never read
    y, _ = hb.mttkrp(h, [None, f[1], f[2]], 0)
    assert y.shape == (5, 2)


def test_foreign_schedule_rejected(hb, rng):
    i1, v1 = _rand(rng, (10, 8, 8), 200)
    i2, v2 = _rand(rng, (10, 8, 8), 100)
    cfg = hb.SplitConfig()
    c1 = hb.build_csf(hb.CooTensor((10, 8, 8), i1, v1), (0, 1, 2))
    c2 = hb.build_csf(hb.CooTensor((10, 8, 8), i2, v2), (0, 1, 2))
    sched = hb.assign_slice_blocks(c1, cfg)
    with pytest.raises(ValueError):
        sched.validate_for(c2)
    f = [np.ones((d, 4)) for d in (10, 8, 8)]
    with pytest.raises(ValueError):
        hb.mttkrp_scheduled(c2, sched, f, 0)


def test_host_built_schedule_and_units(hb, rng):
    idx, vals = _rand(rng, (6, 20, 30), 500)
    t = hb.CooTensor((6, 20, 30), idx, vals)
    cfg = hb.SplitConfig(4, 32, 32)
    c = hb.split_fibers(hb.build_csf(t, (0, 1, 2)), cfg)
    s = hb.assign_slice_blocks(c, cfg)
    host = hb.BlockSchedule(units=s.units, multiplicities=s.multiplicities,
                            num_slices=s.num_slices, num_fibers=s.num_fibers)
    host.validate_for(c)
    f = [rng.random((d, 32)) for d in (6, 20, 30)]
    a, ka = hb.mttkrp_scheduled(c, s, f, 0)
    b, kb = hb.mttkrp_scheduled(c, host, f, 0)
    assert np.allclose(a, b, rtol=1e-6) and ka == kb
    assert all(isinstance(u, hb.ScheduleUnit) for u in s.units)
    bad = hb.BlockSchedule(units=s.units[1:], multiplicities=s.multiplicities,
                           num_slices=s.num_slices, num_fibers=s.num_fibers)
    with pytest.raises(ValueError):
        bad.validate_for(c)


# device tensors ------------------------------------------------------------
def test_device_tensor_inputs(hb, rng):
    import torch

    idx, vals = _rand(rng, (30, 20, 10), 800)
    t_host = hb.CooTensor((30, 20, 10), idx, vals)
    t_dev = hb.CooTensor((30, 20, 10), torch.from_numpy(idx.astype(np.int64)).cuda(),
                         torch.from_numpy(vals).cuda())
    assert t_dev == t_host
    f = [torch.rand((d, 32), device="cuda") for d in (30, 20, 10)]
    fh = [x.double().cpu().numpy() for x in f]
    for mode in range(3):
        h = hb.build_hbcsf(t_dev, hb.allmode_order(t_dev.dims, mode))
        y, _ = hb.mttkrp(h, f, mode)
        assert y.is_cuda and y.dtype == torch.float32
        yd, _ = hb.mttkrp_device(h, f, mode)
        yh, _ = hb.mttkrp(h, fh, mode)
        assert row_dev(y.double().cpu().numpy(), yh) <= 1e-6
        assert row_dev(yd.double().cpu().numpy(), yh) <= 1e-6


def test_canonicalize_merges_duplicates_on_device(hb, rng):
    idx = rng.integers(0, 4, size=(3000, 3)).astype(np.uint32)
    vals = rng.standard_normal(3000)
    idx = np.vstack([idx, [[5, 5, 5], [5, 5, 5]]]).astype(np.uint32)
    vals = np.concatenate([vals, [0.25, -0.25]])  # cancels exactly -> dropped
    ref_i, ref_v = P.canonical(idx, vals)
    c = hb.canonicalize(hb.CooTensor((6, 6, 6), idx, vals))
    assert np.array_equal(c.indices, ref_i) and c.values.tobytes() == ref_v.tobytes()
    assert not ((c.indices == 5).all(axis=1)).any()


# power-law tensors: heavy-slice chunking, all buckets, wide keys ---------
@pytest.mark.parametrize("shape,nnz", [((300, 5000, 2000), 400_000), ((2000, 300000, 30000), 300_000)])
def test_powerlaw_parity_with_oracle(hb, shape, nnz):
    rng = np.random.default_rng(4)
    idx, vals = _powerlaw(rng, shape, nnz)
    t = hb.CooTensor(shape, idx, vals, sorted_under=(0, 1, 2))
    f = [rng.random((d, 32)).astype(np.float32).astype(np.float64) for d in shape]
    for mode in range(3):
        mo = hb.allmode_order(shape, mode)
        h = hb.build_hbcsf(t, mo)
        ref = P.hbcsf(idx, vals, shape, mo)
        assert np.array_equal(h.coo_part.indices, ref["coo"][0])
        assert np.array_equal(h.csl_part.slice_ptr, ref["csl"]["slice_ptr"])
        assert np.array_equal(h.csl_part.rest_idx, ref["csl"]["rest_idx"])
        for d in range(2):
            assert np.array_equal(h.csf_part.ptrs[d], ref["csf"]["ptrs"][d])
            assert np.array_equal(h.csf_part.idxs[d], ref["csf"]["idxs"][d])
        hs = hb.split_fibers(h, hb.SplitConfig())
        refs = P.split_hbcsf(ref, 128)
        assert np.array_equal(hs.csf_part.ptrs[1], refs["csf"]["ptrs"][1])
        sched = hb.assign_slice_blocks(hs.csf_part, hb.SplitConfig())
        units, mult = P.block_schedule(refs["csf"], 512)
        assert np.array_equal(sched.units_array(), units)
        assert np.array_equal(sched.multiplicities, mult)
        yr, kr = P.mttkrp_hbcsf(ref, f, mode)
        y, ops = hb.mttkrp_hbcsf(h, f, mode)
        assert row_dev(y, yr) <= TOL and (ops.muls, ops.adds) == kr
        y2, _ = hb.mttkrp_hbcsf(hs, f, mode)
        assert row_dev(y2, yr) <= TOL
        y3, _ = hb.mttkrp_hbcsf(hs, f, mode, schedule=sched)
        assert row_dev(y3, yr) <= TOL


def test_linearity_and_repeatability(hb):
    rng = np.random.default_rng(9)
    shape = (500, 4000, 3000)
    idx, vals = _powerlaw(rng, shape, 200_000)
    f = [rng.random((d, 32)) for d in shape]
    t1 = hb.CooTensor(shape, idx, vals, sorted_under=(0, 1, 2))
    t2 = hb.CooTensor(shape, idx, 2.0 * vals, sorted_under=(0, 1, 2))
    for mode in range(3):
        mo = hb.allmode_order(shape, mode)
        h1, h2 = hb.build_hbcsf(t1, mo), hb.build_hbcsf(t2, mo)
        a, _ = hb.mttkrp(h1, f, mode)
        b, _ = hb.mttkrp(h2, f, mode)
        # exact up to the run-to-run order of split-slice red.global.add
        assert row_dev(b, 2.0 * a) <= 1e-5
        a2, _ = hb.mttkrp(h1, f, mode)  # the plan is reused; the workspace self-cleans
        assert row_dev(a2, a) <= 1e-5


def test_pinned_host_factors_match_numpy(hb, rng):
    """Page-locked fp32 torch factors take the direct-copy path; results match
    the NumPy path and non-finite entries still raise ValueError."""
    import torch

    idx, vals = _powerlaw(rng, (40, 30, 50), 3000)
    t = hb.CooTensor((40, 30, 50), idx, vals)
    f64 = [rng.random((d, 32)).astype(np.float32).astype(np.float64) for d in (40, 30, 50)]
    pinned = [torch.from_numpy(f).float().pin_memory() for f in f64]
    for mode in range(3):
        h = hb.build_hbcsf(t, hb.allmode_order(t.dims, mode))
        y0, _ = hb.mttkrp_hbcsf(h, f64, mode)
        y1, _ = hb.mttkrp_hbcsf(h, pinned, mode)
        assert isinstance(y1, np.ndarray) and y1.dtype == np.float64
        assert np.array_equal(y0, y1)
    bad = [p.clone().pin_memory() for p in pinned]
    bad[2][3, 4] = float("nan")
    h = hb.build_hbcsf(t, hb.allmode_order(t.dims, 0))
    with pytest.raises(ValueError):
        hb.mttkrp_hbcsf(h, bad, 0)
    # returned rows own their memory: a later call does not overwrite them
    y_a, _ = hb.mttkrp_hbcsf(h, pinned, 0)
    keep = y_a.copy()
    hb.mttkrp_hbcsf(h, [2 * p for p in pinned], 0)
    assert np.array_equal(y_a, keep)


@pytest.mark.parametrize("n", [0, 1, 3, 4, 5, 37, 4096 + 3, 1 << 20])
@pytest.mark.parametrize("offset", [0, 1, 2, 3])
def test_nonfinite_scan(n, offset):
    """hbk_nonfinite_f32 over unaligned heads, float4 bodies and tails: a NaN
    or Inf at the first, a middle and the last position is found, clean
    buffers are not flagged; several buffers in one launch."""
    import ctypes as C

    import torch

    from paper_1904_03329_b200 import _native as N
    from paper_1904_03329_b200.kernels import _nonfinite_flags

    base = torch.rand(n + offset + 8, device="cuda")
    view = base[offset: offset + n]
    clean = torch.rand(777, device="cuda")
    assert _nonfinite_flags(torch, [view, clean]).tolist() == [0, 0]
    for pos in sorted({0, n // 2, n - 1}) if n else []:
        for bad in (float("nan"), float("inf"), float("-inf")):
            v = base.clone()[offset: offset + n]
            v[pos] = bad
            assert _nonfinite_flags(torch, [clean, v, clean]).tolist() == [0, 1, 0]
    # neighbours outside the buffer are not read
    base[:offset] = float("nan")
    base[offset + n:] = float("nan")
    assert _nonfinite_flags(torch, [view]).tolist() == [0]
    with pytest.raises(ValueError):
        N.call("hbk_nonfinite_f32", None, None, 9, None, N.stream_ptr())


@pytest.mark.parametrize("block_mb", ["0.002", "0.0005"])
@pytest.mark.parametrize("rank", [32, 16, 64])
def test_csl_b_row_blocking_parity(hb, rng, block_mb, rank, monkeypatch):
    """The blocked CSL layout (block-major virtual slices, rows accumulated
    with atomics into the zeroed output) gives the oracle's rows, also into a
    dirty output buffer, for R = 32 and the multi-pass ranks.  Tiny blocks
    force many segments per slice and chunked long segments."""
    import torch

    from paper_1904_03329_b200.kernels import mttkrp_device, plan_for

    monkeypatch.setenv("HBK_CSL_BLOCK_MB", block_mb)
    monkeypatch.setenv("HBK_CSL_AS_CSF", "0")  # the CSL kernel itself
    dims = (60, 500, 400)
    # CSL-dominated: distinct (j, k) per slice, so every fiber is a singleton;
    # slice 0 is long (chunked virtual slices)
    n = 6000
    i = np.concatenate([rng.integers(0, 60, n), np.zeros(1500, np.int64)])
    j = rng.integers(0, 500, n + 1500)
    k = rng.integers(0, 400, n + 1500)
    idx = np.stack([i, j, k], 1).astype(np.uint32)
    idx, vals = P.canonical(idx, rng.uniform(0.1, 1.0, n + 1500))
    t = hb.CooTensor(dims, idx, vals)
    f = [rng.random((d, rank)).astype(np.float32).astype(np.float64) for d in dims]
    fd = [torch.from_numpy(x).float().cuda() for x in f]
    for mode in range(3):
        mo = hb.allmode_order(dims, mode)
        h = hb.build_hbcsf(t, mo)
        pl = plan_for(h, mode, rank)
        if h.csl_part.nnz and dims[mo[1]] * 4 * min(rank, 32) > float(block_mb) * 1e6:
            assert pl.info.csl_blocks > 1
        ref, _ = P.mttkrp_hbcsf(P.hbcsf(idx, vals, dims, mo), f, mode)
        y, _ = hb.mttkrp_hbcsf(h, f, mode)
        assert P.row_deviation(y, ref) <= 1e-4
        out = torch.full((dims[mode], rank), 3.0, device="cuda")
        for _ in range(2):  # repeated executions into the same (dirty) buffer
            mttkrp_device(h, fd, mode, out=out)
        assert P.row_deviation(out.double().cpu().numpy(), ref) <= 1e-4
        # fp64 through the same blocked layout (block-major fp64 value stream)
        f64 = [torch.from_numpy(x).cuda() for x in f]
        out64 = torch.full((dims[mode], rank), 3.0, dtype=torch.float64, device="cuda")
        for _ in range(2):
            mttkrp_device(h, f64, mode, out=out64)
        assert P.row_deviation(out64.cpu().numpy(), ref) <= 1e-12


def test_execute_captures_into_cuda_graph(hb, rng):
    """A plan's execute (bucket kernels on forked streams) is capturable into
    a CUDA graph; replays reproduce the eager result for updated factors."""
    import torch

    from paper_1904_03329_b200.kernels import mttkrp_device

    idx, vals = _powerlaw(rng, (300, 200, 400), 60000)
    t = hb.CooTensor((300, 200, 400), idx, vals)
    h = hb.split_fibers(hb.build_hbcsf(t, hb.allmode_order(t.dims, 0)), hb.SplitConfig())
    f = [torch.rand((d, 32), device="cuda") for d in t.dims]
    out = torch.empty((300, 32), device="cuda")
    mttkrp_device(h, f, 0, out=out)  # plan built outside the capture
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        mttkrp_device(h, f, 0, out=out)
    for _ in range(3):
        for x in f:
            x.copy_(torch.rand_like(x))
        g.replay()
        torch.cuda.synchronize()
        ref, _ = mttkrp_device(h, f, 0)
        assert row_dev(out.double().cpu().numpy(), ref.double().cpu().numpy()) <= 1e-5


def test_skip_unowned_rows_and_owned_rows_list(hb, rng):
    """hbk_plan_rows lists exactly the rows with nonzeros; an execute with
    HBK_EXEC_SKIP_UNOWNED writes those rows as the plain execute does and
    leaves every other row untouched."""
    import torch

    from paper_1904_03329_b200.kernels import mttkrp_device, plan_for

    dims = (20000, 60, 80)  # Zipf rows: many of the 20000 stay empty
    idx, vals = _powerlaw(rng, dims, 20000)
    t = hb.CooTensor(dims, idx, vals)
    h = hb.build_hbcsf(t, hb.allmode_order(dims, 0))
    owned = plan_for(h, 0, 32).owned_rows()
    assert owned.tolist() == sorted(set(int(i) for i in idx[:, 0]))
    f = [torch.rand((d, 32), device="cuda") for d in dims]
    full, _ = mttkrp_device(h, f, 0)
    out = torch.full((dims[0], 32), 3.0, device="cuda")
    mttkrp_device(h, f, 0, out=out, skip_unowned=True)
    mask = torch.zeros(dims[0], dtype=torch.bool, device="cuda")
    mask[owned.long()] = True
    assert torch.equal(out[mask], full[mask])
    assert bool((out[~mask] == 3.0).all()) and int((~mask).sum()) > 0


@pytest.mark.parametrize("nnz", [6000, 40000])
def test_csl_slices_through_csf_kernels(hb, rng, nnz, monkeypatch):
    """HB-CSF plans may run their CSL slices as singleton-fiber CSF slices
    (HBK_CSL_AS_CSF; automatic for heavy CSL slices): same rows as the CSL
    kernel and the oracle, same OpCount, for HB-CSF and standalone CSL."""
    dims = (60, 5000, 4000)
    per = nnz // 60  # distinct j within a slice: every fiber is a singleton (CSL)
    i = np.repeat(np.arange(60), per)
    j = np.concatenate([rng.choice(5000, per, replace=False) for _ in range(60)])
    k = rng.integers(0, 4000, 60 * per)
    idx = np.stack([i, j, k], 1).astype(np.uint32)
    idx, vals = P.canonical(idx, rng.uniform(0.1, 1.0, 60 * per))
    t = hb.CooTensor(dims, idx, vals)
    f = [rng.random((d, 32)).astype(np.float32).astype(np.float64) for d in dims]
    ref = loops.mttkrp_entries(idx, vals, dims, f, 0)
    outs = {}
    for flag in ("0", "1"):
        monkeypatch.setenv("HBK_CSL_AS_CSF", flag)
        h = hb.build_hbcsf(t, (0, 1, 2))  # fresh rep: plans are cached per rep
        assert h.csl_part.nnz > 0
        y, ops = hb.mttkrp_hbcsf(h, f, 0)
        y2, ops2 = hb.mttkrp_csl(h.csl_part, f, 0)
        assert row_dev(y, ref) <= TOL
        outs[flag] = (y, (ops.muls, ops.adds), y2, (ops2.muls, ops2.adds))
    assert row_dev(outs["1"][0], outs["0"][0]) <= 1e-5
    assert row_dev(outs["1"][2], outs["0"][2]) <= 1e-5
    assert outs["1"][1] == outs["0"][1] and outs["1"][3] == outs["0"][3]


def test_concurrent_calls_on_one_plan_are_ordered(hb, rng):
    """executions of one plan share its task counters and
    split-slice accumulators.  Calls on one rep from several host threads on
    distinct streams must each produce the full result (libhbk orders them
    on the device), like the reference's mttkrp, which is safe to call
    concurrently."""
    import threading

    import torch

    from paper_1904_03329_b200.kernels import mttkrp_device

    dims = (60, 500, 800)
    idx, vals = _powerlaw(rng, dims, 200000)  # heavy slices: split-slice accumulators
    t = hb.CooTensor(dims, idx, vals)
    h = hb.split_fibers(hb.build_hbcsf(t, hb.allmode_order(dims, 0)), hb.SplitConfig())
    f = [torch.rand((d, 32), device="cuda") for d in dims]
    ref, _ = mttkrp_device(h, f, 0)
    ref = ref.double().cpu().numpy()
    streams = [torch.cuda.Stream() for _ in range(4)]
    outs = [[torch.empty((dims[0], 32), device="cuda") for _ in range(6)] for _ in streams]
    errors = []

    def work(i):
        try:
            with torch.cuda.stream(streams[i]):
                for o in outs[i]:
                    mttkrp_device(h, f, 0, out=o)
        except Exception as e:  # pragma: no cover - surfaced below
            errors.append(e)

    ths = [threading.Thread(target=work, args=(i,)) for i in range(len(streams))]
    for th in ths:
        th.start()
    for th in ths:
        th.join()
    torch.cuda.synchronize()
    assert not errors, errors
    for per_stream in outs:
        for o in per_stream:
            assert row_dev(o.double().cpu().numpy(), ref) <= 1e-5
    # host-array calls from threads (the reference calling convention)
    fh = [x.double().cpu().numpy() for x in f]
    res = [None] * 4

    def host_call(i):
        res[i] = hb.mttkrp_hbcsf(h, fh, 0)[0]

    ths = [threading.Thread(target=host_call, args=(i,)) for i in range(4)]
    for th in ths:
        th.start()
    for th in ths:
        th.join()
    for y in res:
        assert row_dev(y, ref) <= 1e-5


def test_finite_factor_beyond_fp32_range_is_rejected(hb, rng):
    """a finite float64 factor with |x| > FLT_MAX would reach the
    fp32 kernel as inf; the host calling convention raises instead (the fp64
    kernel takes it)."""
    idx, vals = _powerlaw(rng, (30, 20, 40), 2000)
    t = hb.CooTensor((30, 20, 40), idx, vals)
    h = hb.build_hbcsf(t, (0, 1, 2))
    f = [rng.random((d, 32)) for d in t.dims]
    f[2][3, 5] = 1e39
    with pytest.raises(ValueError, match="float32 range"):
        hb.mttkrp_hbcsf(h, f, 0)
    y, _ = hb.mttkrp_hbcsf(h, f, 0, precision="fp64")
    assert np.isfinite(y).all()


@pytest.mark.parametrize("n", [0, 1, 7, 8, 9, 65536 - 3, 65536, 65536 * 3 + 5])
@pytest.mark.parametrize("offset", [0, 1, 5])
@pytest.mark.parametrize("dst", ["f32", "f64"])
def test_stage_f64_to_f32(n, offset, dst):
    """hbk_stage_f64_to_f32 (the host calling convention's float64 -> fp32
    upload): every element round-to-nearest exactly as NumPy's astype, over
    unaligned staging heads, 8-wide bodies, tails and several chunks; the
    non-finite / beyond-fp32-range flag per factor; several factors per call."""
    import ctypes as C

    import torch

    from paper_1904_03329_b200 import _native as N

    rng = np.random.default_rng(n + offset)
    srcs = [rng.standard_normal(n) * 10.0 ** rng.integers(-40, 40, n) if n else np.zeros(0),
            rng.random(777)]
    tdt, ndt = (torch.float32, np.float32) if dst == "f32" else (torch.float64, np.float64)
    stage_base = [torch.empty(len(s) + offset + 8, dtype=tdt, pin_memory=True) for s in srcs]
    stages = [b[offset: offset + len(s)] for b, s in zip(stage_base, srcs)]
    devs = [torch.full((len(s) + 1,), -7.0, dtype=tdt, device="cuda") for s in srcs]

    def run(arrs):
        k = len(arrs)
        flags = (C.c_int32 * k)()
        N.call(f"hbk_stage_f64_to_{dst}", (C.c_void_p * k)(*[a.ctypes.data for a in arrs]),
               (C.c_int64 * k)(*[a.size for a in arrs]), k,
               (C.c_void_p * k)(*[s.data_ptr() for s in stages]),
               (C.c_void_p * k)(*[d.data_ptr() for d in devs]), flags, N.stream_ptr())
        torch.cuda.synchronize()
        return list(flags)

    with np.errstate(over="ignore"):
        want = [s.astype(ndt) for s in srcs]
    fl = run(srcs)
    ui = np.uint32 if dst == "f32" else np.uint64
    for s, w, d, f in zip(srcs, want, devs, fl):
        got = d[: len(s)].cpu().numpy()
        assert np.array_equal(got.view(ui), w.view(ui))
        assert d[len(s)].item() == -7.0  # nothing written past the end
        assert f == int(not np.isfinite(w).all())
    if n:
        for pos in sorted({0, n // 2, n - 1}):
            for bad in (np.nan, np.inf, -np.inf) + ((1e39,) if dst == "f32" else ()):
                s0 = np.clip(srcs[0], -1e30, 1e30)
                s0[pos] = bad
                assert run([s0, srcs[1]]) == [1, 0]
        assert run([np.clip(srcs[0], -1e30, 1e30), srcs[1]]) == [0, 0]
    with pytest.raises(ValueError):
        N.call(f"hbk_stage_f64_to_{dst}", None, None, 9, None, None, None, N.stream_ptr())


def test_host_factor_errors_raised_before_launch(hb, rng):
    """A NaN in a NumPy float64 factor is reported by the staging pass before
    the kernel runs (kernels.py:82-86), the plan stays usable."""
    idx, vals = _powerlaw(rng, (30, 20, 40), 2000)
    t = hb.CooTensor((30, 20, 40), idx, vals)
    h = hb.build_hbcsf(t, (0, 1, 2))
    f = [rng.random((d, 32)) for d in t.dims]
    ok, _ = hb.mttkrp_hbcsf(h, f, 0)
    bad = [x.copy() for x in f]
    bad[1][4, 7] = np.nan
    with pytest.raises(ValueError, match="non-finite"):
        hb.mttkrp_hbcsf(h, bad, 0)
    again, _ = hb.mttkrp_hbcsf(h, f, 0)
    assert np.array_equal(ok, again)


def test_fiber_histogram_matches_csf(hb, rng):
    """hbk_coo_fiber_histogram: distinct (slice, mid) pairs per slice equal the
    per-slice fiber counts of the CSF tree in that order (formats.py:143-162),
    for every mode and both mid modes; partition_costs = nnz + fibers + ROW_COST."""
    from paper_1904_03329_b200 import shard

    dims = (70, 50, 90)
    idx, vals = _powerlaw(rng, dims, 8000)
    t = hb.CooTensor(dims, idx, vals)
    for mode in range(3):
        for mid in (d for d in range(3) if d != mode):
            leaf = 3 - mode - mid
            c = hb.build_csf(t, (mode, mid, leaf))
            want = np.zeros(dims[mode], np.int64)
            want[c.idxs[0]] = np.diff(c.ptrs[0])
            got = shard.fiber_histogram(t, mode, mid).cpu().numpy()
            assert np.array_equal(got, want)
        nnz = np.bincount(idx[:, mode].astype(np.int64), minlength=dims[mode])
        mid = hb.allmode_order(dims, mode)[1]
        fib = shard.fiber_histogram(t, mode, mid).cpu().numpy()
        cost = shard.partition_costs(t, mode).cpu().numpy()
        assert np.array_equal(cost, nnz + fib + shard.ROW_COST)


@pytest.mark.parametrize("block_mb,minnz", [("0.002", "8"), ("0.0005", "64"), ("0.004", "1")])
@pytest.mark.parametrize("rank", [32, 16, 64])
def test_leaf_blocked_heavy_slices_parity(hb, rng, block_mb, minnz, rank, monkeypatch):
    """Leaf-blocked heavy slices (csf_block_view + accumulating sub-plan):
    the oracle's rows for every mode, R = 32 and multi-pass ranks, into a
    dirty output buffer; the fp64 (generic) kernel and the OpCount stay the
    reference's; owned rows unchanged; skip-unowned keeps heavy rows."""
    import torch

    from paper_1904_03329_b200.kernels import mttkrp_device, plan_for

    monkeypatch.setenv("HBK_LEAF_BLOCK_MB", block_mb)
    monkeypatch.setenv("HBK_LEAF_MIN", minnz)
    dims = (80, 60, 500)
    idx, vals = _powerlaw(rng, dims, 12000)
    # a few very heavy slices (heavy layout inside the blocked view) and a COO tail
    extra = np.stack([np.zeros(3000, np.int64), rng.integers(0, 60, 3000), rng.integers(0, 500, 3000)], 1)
    idx, vals = P.canonical(np.vstack([idx.astype(np.int64), extra]).astype(np.uint32),
                            np.concatenate([vals, rng.uniform(0.1, 1.0, 3000)]))
    t = hb.CooTensor(dims, idx, vals)
    f = [rng.random((d, rank)).astype(np.float32).astype(np.float64) for d in dims]
    fd = [torch.from_numpy(x).float().cuda() for x in f]
    for mode in range(3):
        mo = hb.allmode_order(dims, mode)
        h = hb.split_fibers(hb.build_hbcsf(t, mo), hb.SplitConfig(fiber_threshold=16))
        pl = plan_for(h, mode, rank)
        ref_h = P.split_hbcsf(P.hbcsf(idx, vals, dims, mo), 16)
        ref, ops = P.mttkrp_hbcsf(ref_h, f, mode)
        y, oc = hb.mttkrp_hbcsf(h, f, mode)
        assert P.row_deviation(y, ref) <= 1e-4
        assert (oc.muls, oc.adds) == tuple(ops)
        if dims[mo[2]] * 4 * min(rank, 32) > float(block_mb) * 1e6:
            assert pl.info.leaf_blocks > 1 and pl.info.leaf_blocked_nnz > 0
        out = torch.full((dims[mode], rank), 3.0, device="cuda")
        for _ in range(2):
            mttkrp_device(h, fd, mode, out=out)
        assert P.row_deviation(out.double().cpu().numpy(), ref) <= 1e-4
        y64, _ = hb.mttkrp_hbcsf(h, f, mode, precision="fp64")
        assert P.row_deviation(y64, ref) <= 1e-12
        out64 = torch.full((dims[mode], rank), 3.0, dtype=torch.float64, device="cuda")
        for _ in range(2):  # the fp64 fast path through the blocked pair, dirty buffer
            mttkrp_device(h, [x.double() for x in fd], mode, out=out64)
        assert P.row_deviation(out64.cpu().numpy(), ref) <= 1e-12
        owned = pl.owned_rows().cpu().numpy()
        want = np.nonzero(np.bincount(idx[:, mode].astype(np.int64), minlength=dims[mode]))[0]
        assert np.array_equal(np.sort(owned), want)
        out.fill_(7.0)
        mttkrp_device(h, fd, mode, out=out, skip_unowned=True)
        got = out.double().cpu().numpy()
        assert P.row_deviation(got[want], ref[want]) <= 1e-4


@pytest.mark.parametrize("rank", [32, 16, 36])
def test_fp64_fast_path_matches_generic_and_oracle(hb, rng, rank, monkeypatch):
    """precision="fp64" runs the fast kernels on double2 lanes (fp64 value
    streams, 16-column passes) for every bucket kind; rows agree with the
    generic fp64 kernel to 1e-13 and with the loop oracle to 1e-12."""
    from paper_1904_03329_b200.kernels import plan_for

    dims = (40, 30, 500)
    idx, vals = _powerlaw(rng, dims, 6000)
    heavy = np.stack([np.zeros(2500, np.int64), rng.integers(0, 30, 2500), rng.integers(0, 500, 2500)], 1)
    idx, vals = P.canonical(np.vstack([idx.astype(np.int64), heavy]).astype(np.uint32),
                            np.concatenate([vals, rng.uniform(0.1, 1.0, 2500)]))
    t = hb.CooTensor(dims, idx, vals)
    f = [rng.standard_normal((d, rank)) for d in dims]
    for mode in range(3):
        mo = hb.allmode_order(dims, mode)
        h = hb.split_fibers(hb.build_hbcsf(t, mo), hb.SplitConfig(fiber_threshold=16))
        yf, ops = hb.mttkrp_hbcsf(h, f, mode, precision="fp64")
        ref, rops = P.mttkrp_hbcsf(P.split_hbcsf(P.hbcsf(idx, vals, dims, mo), 16), f, mode)
        assert P.row_deviation(yf, ref) <= 1e-12
        assert (ops.muls, ops.adds) == tuple(rops)
        monkeypatch.setenv("HBK_F64_GENERIC", "1")
        hg = hb.split_fibers(hb.build_hbcsf(t, mo), hb.SplitConfig(fiber_threshold=16))
        yg, _ = hb.mttkrp_hbcsf(hg, f, mode, precision="fp64")
        monkeypatch.delenv("HBK_F64_GENERIC")
        assert P.row_deviation(yf, yg) <= 1e-13
        assert plan_for(h, mode, rank).info.fast_path
