"""compute_stats / imbalance_metrics against a NumPy
restatement of the reference's group counting (coo.py:281-325,
balance.py:210-227), including duplicate coordinates and split trees."""
from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _group_counts(idx, mo, ncols):
    keys = idx[:, list(mo)]
    order = np.lexsort([keys[:, c] for c in reversed(range(keys.shape[1]))])
    cols = keys[order][:, :ncols]
    new = np.empty(len(cols), dtype=bool)
    new[0] = True
    np.not_equal(cols[1:], cols[:-1]).any(axis=1, out=new[1:])
    starts = np.flatnonzero(new)
    return np.diff(np.append(starts, len(cols)))


@pytest.mark.parametrize("mo", [(0, 1, 2), (2, 0, 1), (1, 2, 0)])
def test_compute_stats_matches_reference_counting(mo):
    import paper_1904_03329_b200 as hb

    rng = np.random.default_rng(3)
    dims = (30, 20, 40)
    idx = np.stack([rng.integers(0, d, 5000) for d in dims], 1).astype(np.uint32)
    idx[:50] = idx[50:100]  # duplicates count as distinct entries
    vals = rng.random(5000)
    s = hb.compute_stats(hb.CooTensor(dims, idx, vals), mo)
    sl = _group_counts(idx, mo, 1)
    fb = _group_counts(idx, mo, 2)
    assert s.mode_order == mo and s.nnz == 5000
    assert s.density == pytest.approx(5000 / (30 * 20 * 40))
    assert (s.slice_count, s.fiber_count) == (len(sl), len(fb))
    assert s.max_nnz_per_slice == sl.max() and s.max_nnz_per_fiber == fb.max()
    assert s.mean_nnz_per_slice == pytest.approx(sl.mean(), rel=1e-12)
    assert s.stddev_nnz_per_slice == pytest.approx(sl.std(), rel=1e-12)
    assert s.mean_nnz_per_fiber == pytest.approx(fb.mean(), rel=1e-12)
    assert s.stddev_nnz_per_fiber == pytest.approx(fb.std(), rel=1e-12)
    assert s.to_dict()["mode_order"] == list(mo)


def test_imbalance_metrics_split_tree():
    import paper_1904_03329_b200 as hb

    rng = np.random.default_rng(4)
    dims = (8, 6, 300)
    idx = np.stack([rng.integers(0, d, 3000) for d in dims], 1).astype(np.uint32)
    t = hb.canonicalize(hb.CooTensor(dims, idx, rng.random(3000)))
    c = hb.split_fibers(hb.build_csf(t, (0, 1, 2)), hb.SplitConfig(fiber_threshold=4, block_size=64))
    m = hb.imbalance_metrics(c)
    fs = np.diff(c.ptrs[1])
    ss = np.array([c.leaf_offsets()[i + 1] - c.leaf_offsets()[i] for i in range(c.num_slices)])
    assert (m.slices, m.fibers, m.nnz) == (c.num_slices, c.num_fibers, c.nnz)
    assert m.max_nnz_per_fiber == fs.max() <= 4
    assert m.mean_nnz_per_fiber == pytest.approx(fs.mean())
    assert m.stddev_nnz_per_slice == pytest.approx(ss.std())
    empty = hb.imbalance_metrics(hb.build_csf(hb.CooTensor(dims, np.zeros((0, 3), np.uint32), []), (0, 1, 2)))
    assert empty.nnz == 0 and empty.max_nnz_per_slice == 0


FIG = np.array([[0, 0, 0], [1, 0, 0], [1, 1, 1], [1, 2, 2], [2, 1, 0], [2, 1, 1], [2, 1, 2], [2, 1, 3]],
               dtype=np.uint32)  # tests/helpers.py FIG tensor (helpers.py:18-28 of the reference), 0-based


def test_storage_and_census_walkthrough():
    """The reference's storage / census known answers (test_formats.py:88-91,
    116, 156-163) through the device reductions."""
    import paper_1904_03329_b200 as hb

    t = hb.canonicalize(hb.CooTensor((3, 3, 4), FIG, np.arange(1.0, 9.0)))
    assert hb.storage_words(t).index_words == 24
    c = hb.build_csf(t, (0, 1, 2))
    assert hb.storage_words(c).index_words == 24
    assert hb.slice_census(c) == {"coo": 1, "csl": 1, "csf": 1}
    h = hb.build_hbcsf(t, (0, 1, 2))
    assert hb.slice_census(h) == {"coo": 1, "csl": 1, "csf": 1}
    rep = hb.storage_words(h)
    assert rep.index_words == 19 and [p.words for p in rep.parts] == [3, 8, 8] and rep.index_bytes == 76
    p = hb.storage_words(t).parts[0]
    assert (p.slices, p.fibers) == (3, 5)


@pytest.mark.parametrize("mo", [(0, 1, 2), (2, 1, 0)])
def test_device_census_and_coo_storage_match_host_counting(mo):
    import paper_1904_03329_b200 as hb

    rng = np.random.default_rng(9)
    dims = (300, 40, 50)
    i0 = np.minimum((rng.pareto(1.0, 8000) * 4).astype(np.int64), dims[0] - 1)
    idx = np.stack([i0, rng.integers(0, dims[1], 8000), rng.integers(0, dims[2], 8000)], 1).astype(np.uint32)
    t = hb.canonicalize(hb.CooTensor(dims, idx, rng.random(8000)))
    c = hb.build_csf(t, mo)
    labels = hb.classify_slices(c)
    census = hb.slice_census(c)
    assert census == {"coo": int((labels == 0).sum()), "csl": int((labels == 1).sum()),
                      "csf": int((labels == 2).sum())}
    if mo[0] == 0:  # the skewed mode: every class occurs
        assert census["coo"] > 0 and census["csl"] > 0 and census["csf"] > 0
    ts = hb.sort_by_mode_order(t, mo)
    p = hb.storage_words(ts).parts[0]
    keys = ts.indices[:, list(mo)]
    assert p.slices == len(np.unique(keys[:, 0]))
    assert p.fibers == len(np.unique(keys[:, :2], axis=0))
