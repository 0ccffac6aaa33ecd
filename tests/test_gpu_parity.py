"""GPU parity: the libhbk path against the reference's golden outputs.

Format arrays (CSF / HB-CSF parts, labels, split arrays, schedules) must be
bit-identical; fp32 MTTKRP outputs within the row metric
max ||y_i - o_i|| / (1 + ||o_i||) <= 1e-4 (BASELINE.json north_star; fp32
storage/accumulation and atomic ordering); OpCounts exact.
"""
from __future__ import annotations

import numpy as np
import pytest

from conftest import golden
from helpers import cases, cfg_blocks, digest, golden_factors, mode_blocks, rank_blocks, row_dev

pytestmark = pytest.mark.gpu

TOL = 1e-4


@pytest.fixture(scope="module")
def hb():
    import paper_1904_03329_b200 as hb

    return hb


def _tree_eq(c, g, prefix, order):
    for d in range(order - 1):
        assert np.array_equal(c.ptrs[d], g[f"{prefix}/ptr{d}"]), f"{prefix}/ptr{d}"
        assert c.ptrs[d].dtype == np.int64
        assert np.array_equal(c.idxs[d], g[f"{prefix}/idx{d}"]), f"{prefix}/idx{d}"
        assert c.idxs[d].dtype == np.uint32


@pytest.mark.parametrize("case", [c[0] for c in cases()])
def test_formats_bit_exact(hb, case):
    g = golden("formats_kernels")
    key, idx, vals, dims = next(c for c in cases() if c[0] == case)
    t = hb.CooTensor(dims, idx, vals)
    for mode, p in mode_blocks(key):
        mo = tuple(int(x) for x in g[f"{p}/mode_order"])
        assert hb.allmode_order(dims, mode) == mo
        c = hb.build_csf(t, mo)
        _tree_eq(c, g, f"{p}/csf", len(dims))
        assert np.array_equal(c.leaf_idx, g[f"{p}/csf/leaf"])
        assert c.values.tobytes() == g[f"{p}/csf/values"].tobytes()
        assert np.array_equal(hb.classify_slices(c), g[f"{p}/labels"])
        h = hb.build_hbcsf(t, mo)
        assert np.array_equal(h.coo_part.indices, g[f"{p}/hb/coo/indices"])
        assert h.coo_part.values.tobytes() == g[f"{p}/hb/coo/values"].tobytes()
        assert h.coo_part.sorted_under == mo
        assert np.array_equal(h.csl_part.slice_ptr, g[f"{p}/hb/csl/slice_ptr"])
        assert np.array_equal(h.csl_part.slice_idx, g[f"{p}/hb/csl/slice_idx"])
        assert np.array_equal(h.csl_part.rest_idx, g[f"{p}/hb/csl/rest_idx"])
        assert h.csl_part.values.tobytes() == g[f"{p}/hb/csl/values"].tobytes()
        _tree_eq(h.csf_part, g, f"{p}/hb/csf", len(dims))
        assert np.array_equal(h.csf_part.leaf_idx, g[f"{p}/hb/csf/leaf"])
        for _, q, (tau, bs, ws) in cfg_blocks(p):
            cfg = hb.SplitConfig(tau, bs, ws)
            hs = hb.split_fibers(h, cfg)
            assert hs.coo_part is h.coo_part and hs.csl_part is h.csl_part
            assert (hs.csf_part is h.csf_part) == bool(g[f"{q}/split_is_noop"])
            _tree_eq(hs.csf_part, g, f"{q}/split", len(dims))
            sched = hb.assign_slice_blocks(hs.csf_part, cfg)
            assert np.array_equal(sched.units_array(), g[f"{q}/units"])
            assert np.array_equal(sched.multiplicities, g[f"{q}/mult"])
            sched.validate_for(hs.csf_part)
            cs = hb.split_fibers(c, cfg)
            assert np.array_equal(cs.ptrs[-1], g[f"{q}/csfsplit/ptr{len(dims) - 2}"])
            fs = hb.assign_slice_blocks(cs, cfg)
            assert np.array_equal(fs.units_array(), g[f"{q}/csfsplit/units"])


@pytest.mark.parametrize("case", [c[0] for c in cases()])
def test_mttkrp_all_variants(hb, case):
    g = golden("formats_kernels")
    key, idx, vals, dims = next(c for c in cases() if c[0] == case)
    t = hb.CooTensor(dims, idx, vals)
    for mode, p in mode_blocks(key):
        mo = tuple(int(x) for x in g[f"{p}/mode_order"])
        h = hb.build_hbcsf(t, mo)
        c = hb.build_csf(t, mo)
        for _, q, (tau, bs, ws) in cfg_blocks(p):
            cfg = hb.SplitConfig(tau, bs, ws)
            hs = hb.split_fibers(h, cfg)
            sched = hb.assign_slice_blocks(hs.csf_part, cfg)
            cs = hb.split_fibers(c, cfg)
            fsched = hb.assign_slice_blocks(cs, cfg)
            for r, fr in rank_blocks(q):
                f = golden_factors(fr, dims, r)
                ref = g[f"{fr}/y"]
                runs = {
                    "hbcsf": hb.mttkrp_hbcsf(h, f, mode),
                    "hbsched": hb.mttkrp_hbcsf(hs, f, mode, schedule=sched),
                    "csf": hb.mttkrp_csf(c, f, mode),
                    "sched": hb.mttkrp_scheduled(cs, fsched, f, mode),
                    "coo": hb.mttkrp_coo(t, f, mode),
                }
                for name, (y, ops) in runs.items():
                    assert y.dtype == np.float64 and y.shape == ref.shape
                    dev = row_dev(y, ref)
                    assert dev <= TOL, (name, r, dev)
                    assert [ops.muls, ops.adds] == g[f"{fr}/ops_{name}"].tolist(), name
                y, ops = hb.mttkrp(hs, f, mode)
                assert row_dev(y, ref) <= TOL
                y, _ = hb.mttkrp(h.csl_part, f, mode)
                y2, _ = hb.mttkrp(h.coo_part, f, mode)
                y3, _ = hb.mttkrp(h.csf_part, f, mode)
                assert row_dev(y + y2 + y3, ref) <= TOL


def test_config1_bit_exact_and_output(hb):
    g = golden("config1")
    dims = tuple(int(d) for d in g["dims"])
    t = hb.CooTensor(dims, g["indices"], g["values"], sorted_under=(0, 1, 2))
    mo = hb.allmode_order(dims, 0)
    cfg = hb.SplitConfig()
    h = hb.build_hbcsf(t, mo)
    hs = hb.split_fibers(h, cfg)
    sched = hb.assign_slice_blocks(hs.csf_part, cfg)
    arrays = {
        "coo/indices": h.coo_part.indices, "coo/values": h.coo_part.values,
        "csl/slice_ptr": h.csl_part.slice_ptr, "csl/slice_idx": h.csl_part.slice_idx,
        "csl/rest_idx": h.csl_part.rest_idx, "csl/values": h.csl_part.values,
        "csf/ptr0": h.csf_part.ptrs[0], "csf/ptr1": h.csf_part.ptrs[1],
        "csf/idx0": h.csf_part.idxs[0], "csf/idx1": h.csf_part.idxs[1],
        "csf/leaf": h.csf_part.leaf_idx, "csf/values": h.csf_part.values,
        "split/ptr0": hs.csf_part.ptrs[0], "split/ptr1": hs.csf_part.ptrs[1],
        "split/idx1": hs.csf_part.idxs[1], "mult": sched.multiplicities,
        "units": sched.units_array(),
    }
    for name, arr in arrays.items():
        assert digest(arr) == str(g[f"sha/{name}"]), name
    census = [h.coo_part.nnz, h.csl_part.num_slices, h.csf_part.num_slices, h.csl_part.nnz,
              h.csf_part.nnz, h.csf_part.num_fibers]
    assert census == g["census"].tolist()
    frng = np.random.default_rng(0)
    f = [frng.random((d, 32)).astype(np.float32).astype(np.float64) for d in dims]
    y, ops = hb.mttkrp_hbcsf(hs, f, 0)
    assert row_dev(y, g["y"]) <= TOL
    assert [ops.muls, ops.adds] == g["ops"].tolist()
    y, ops = hb.mttkrp_hbcsf(hs, f, 0, schedule=sched)
    assert row_dev(y, g["y"]) <= TOL
    assert [ops.muls, ops.adds] == g["ops_sched"].tolist()


def test_canonicalize_bitwise(hb):
    g = golden("canonicalize")
    for key in ("dup_small", "dup_runs", "longrun"):
        idx, vals = g[f"{key}/in_indices"], g[f"{key}/in_values"]
        dims = tuple(int(x) + 1 for x in idx.max(axis=0))
        c = hb.canonicalize(hb.CooTensor(dims, idx, vals))
        assert np.array_equal(c.indices, g[f"{key}/out_indices"])
        assert c.values.tobytes() == g[f"{key}/out_values"].tobytes()
        assert c.sorted_under == (0, 1, 2)


def test_sort_by_mode_order_matches_lexsort(hb, rng):
    from oracle import tenkit_port as P

    dims = (70, 3, 900000)
    idx = np.stack([rng.integers(0, d, 5000) for d in dims], axis=1).astype(np.uint32)
    idx[::7] = idx[3]  # duplicates: stability matters
    vals = rng.random(5000)
    t = hb.CooTensor(dims, idx, vals)
    for mo in [(0, 1, 2), (2, 0, 1), (1, 2, 0)]:
        s = hb.sort_by_mode_order(t, mo)
        ri, rv = P.sort_entries(idx, vals, mo)
        assert np.array_equal(s.indices, ri) and np.array_equal(s.values, rv)
        assert s.sorted_under == mo
        assert hb.sort_by_mode_order(s, mo) is s


def test_wide_keys_sort(hb, rng):
    """Keys wider than 64 bits (flickr/delicious/nell-1 shapes)."""
    from oracle import tenkit_port as P

    dims = (319686, 28153045, 1607191)
    n = 20000
    idx = np.stack([rng.integers(0, d, n) for d in dims], axis=1).astype(np.uint32)
    idx[: n // 2, 0] = 5  # many shared slices
    idx[: n // 4, 1] = 77
    vals = rng.random(n)
    t = hb.CooTensor(dims, idx, vals)
    for mode in range(3):
        mo = hb.allmode_order(dims, mode)
        s = hb.sort_by_mode_order(t, mo)
        ri, _ = P.sort_entries(idx, vals, mo)
        assert np.array_equal(s.indices, ri)
        h = hb.build_hbcsf(t, mo)
        ref = P.hbcsf(idx, vals, dims, mo)
        assert np.array_equal(h.csl_part.slice_ptr, ref["csl"]["slice_ptr"])
        for d in range(2):
            assert np.array_equal(h.csf_part.ptrs[d], ref["csf"]["ptrs"][d])
            assert np.array_equal(h.csf_part.idxs[d], ref["csf"]["idxs"][d])
