"""Host-side logic of the drop-in API that runs without a GPU: argument
validation (same exceptions as the reference), mode orders, split config,
OpCount, the small dense CP-ALS algebra and the shard planner."""
from __future__ import annotations

import numpy as np
import pytest

import paper_1904_03329_b200 as hb
from paper_1904_03329_b200.kernels import _check_factors
from paper_1904_03329_b200.shard import plan_row_ranges


def test_cootensor_validation_matches_reference():
    with pytest.raises(ValueError):
        hb.CooTensor((2, 2), np.zeros((1, 2)), [1.0])
    with pytest.raises(ValueError):
        hb.CooTensor((2, 0, 2), np.zeros((1, 3)), [1.0])
    with pytest.raises(ValueError):
        hb.CooTensor((2, 2, 2), np.zeros((1, 2)), [1.0])
    with pytest.raises(ValueError):
        hb.CooTensor((2, 2, 2), np.zeros((2, 3)), [1.0])
    with pytest.raises(ValueError):
        hb.CooTensor((2, 2, 2), np.array([[0, 0, 2]]), [1.0])
    with pytest.raises(ValueError):
        hb.CooTensor((2, 2, 2), np.zeros((1, 3)), [1.0], sorted_under=(0, 0, 1))
    t = hb.CooTensor((2, 3, 4), np.array([[1, 2, 3]]), [2.5])
    assert t.indices.dtype == np.uint32 and t.values.dtype == np.float64
    assert t.order == 3 and t.nnz == 1
    assert list(t.entries()) == [((1, 2, 3), 2.5)]
    assert t == hb.CooTensor((2, 3, 4), np.array([[1, 2, 3]]), [2.5])


def test_allmode_order_ties():
    assert hb.allmode_order((5, 3, 3, 4), 0) == (0, 1, 2, 3)
    assert hb.allmode_order((5, 3, 3, 4), 2) == (2, 1, 3, 0)
    assert hb.allmode_order((12092, 9184, 28818), 2) == (2, 1, 0)
    assert hb.allmode_order((319686, 28153045, 1607191), 0) == (0, 2, 1)
    with pytest.raises(ValueError):
        hb.allmode_order((3, 3, 3), 3)


def test_split_config_validation():
    with pytest.raises(ValueError):
        hb.SplitConfig(fiber_threshold=0)
    with pytest.raises(ValueError):
        hb.SplitConfig(block_size=0)
    with pytest.raises(ValueError):
        hb.SplitConfig(block_size=100, warp_size=32)
    assert hb.SplitConfig() == hb.SplitConfig(128, 512, 32)


def test_check_factors_errors():
    dims = (3, 4, 5)
    good = [np.zeros((3, 2)), np.zeros((4, 2)), np.zeros((5, 2))]
    assert _check_factors(dims, good, 0) == 2
    with pytest.raises(ValueError):
        _check_factors(dims, good, 3)
    with pytest.raises(ValueError):
        _check_factors(dims, good[:2], 0)
    with pytest.raises(ValueError):
        _check_factors(dims, [good[0], np.zeros((4, 3)), good[2]], 0)
    with pytest.raises(ValueError):
        _check_factors(dims, [good[0], np.zeros((5, 2)), good[2]], 0)
    bad = [good[0], good[1], np.full((5, 2), np.nan)]
    with pytest.raises(ValueError):
        _check_factors(dims, bad, 0)
    # factors[mode] is never inspected (kernels.py:62-66)
    assert _check_factors(dims, [None, good[1], good[2]], 0) == 2


def test_dispatch_rejects_unknown_type():
    with pytest.raises(TypeError):
        hb.mttkrp(object(), [], 0)
    with pytest.raises(TypeError):
        hb.split_fibers(object(), hb.SplitConfig())


def test_opcount_arithmetic():
    a, b = hb.OpCount(3, 4), hb.OpCount(10, 20)
    assert (a + b).total == 37 and (a + b).to_dict() == {"muls": 13, "adds": 24, "total": 37}


def test_dense_cpd_helpers(rng):
    f = rng.standard_normal((7, 3))
    g = hb.gram(f)
    assert np.allclose(g, f.T @ f) and np.array_equal(g, g.T)
    grams = [hb.gram(rng.standard_normal((5, 3))) for _ in range(3)]
    assert np.allclose(hb.hadamard_all_but(grams, 0), grams[1] * grams[2])
    a = rng.standard_normal((6, 4))
    s = a.T @ a
    p = hb.pinv_spsd(s)
    assert np.allclose(s @ p @ s, s, atol=1e-10)
    with pytest.raises(ValueError):
        hb.pinv_spsd(np.array([[1.0, 2.0], [0.0, 1.0]]))
    with pytest.raises(ValueError):
        hb.pinv_spsd(-np.eye(3))


def test_plan_row_ranges_balanced_and_exact():
    counts = np.array([5, 1, 1, 1, 10, 0, 2, 3, 7, 1])
    for parts in (1, 2, 3, 4, 10, 12):
        rr = plan_row_ranges(counts, parts)
        assert len(rr) == parts
        assert rr[0][0] == 0 and rr[-1][1] == len(counts)
        assert all(a[1] == b[0] for a, b in zip(rr[:-1], rr[1:]))
        assert sum(int(counts[lo:hi].sum()) for lo, hi in rr) == counts.sum()
    rng = np.random.default_rng(3)
    c = rng.zipf(1.5, 10000).clip(max=500)
    rr = plan_row_ranges(c, 8)
    loads = [int(c[lo:hi].sum()) for lo, hi in rr]
    assert max(loads) - min(loads) <= 2 * c.max()


def test_refine_row_ranges_equalises_measured_time():
    """Calibration pass: rows whose measured time per cost unit is higher
    (a slow region of the row space) get more weight, so a synthetic 'true
    time' that the static costs mis-model comes out balanced after one pass."""
    from paper_1904_03329_b200.shard import refine_row_ranges

    rng = np.random.default_rng(5)
    costs = rng.integers(1, 50, 20000)
    rate = np.where(np.arange(20000) > 15000, 3.0, 1.0)  # the tail runs 3x slower per unit
    true = costs * rate
    for parts in (2, 4, 8):
        rr = plan_row_ranges(costs, parts)
        t0 = [float(true[lo:hi].sum()) for lo, hi in rr]
        rr2 = refine_row_ranges(costs, rr, t0)
        t1 = [float(true[lo:hi].sum()) for lo, hi in rr2]
        assert rr2[0][0] == 0 and rr2[-1][1] == len(costs)
        assert all(a[1] == b[0] for a, b in zip(rr2[:-1], rr2[1:]))
        assert max(t1) / np.mean(t1) < max(t0) / np.mean(t0)
        assert max(t1) / np.mean(t1) < 1.2
    # float weights and zero-time ranges are accepted
    assert refine_row_ranges(costs, [(0, 10000), (10000, 20000)], [0.0, 1.0])[-1][1] == 20000
