"""Pin the CPU oracle (oracle/tenkit_port.py) to the reference's own outputs.

The golden fixtures were produced by running the reference package
(tests/golden/make_golden.py).  Integer arrays must match exactly, fp64
MTTKRP outputs to 1e-12 (row metric), OpCounts exactly.  CPU only.
"""
from __future__ import annotations

import numpy as np
import pytest

from conftest import golden
from helpers import cases, cfg_blocks, digest, golden_factors, mode_blocks, rank_blocks, row_dev
from oracle import loops
from oracle import tenkit_port as P


def _tree_eq(tree, g, prefix, order):
    for d in range(order - 1):
        assert np.array_equal(tree["ptrs"][d], g[f"{prefix}/ptr{d}"]), f"{prefix}/ptr{d}"
        assert tree["ptrs"][d].dtype == np.int64
        assert np.array_equal(tree["idxs"][d], g[f"{prefix}/idx{d}"]), f"{prefix}/idx{d}"


@pytest.mark.parametrize("case", [c[0] for c in cases()])
def test_oracle_formats_match_reference(case):
    g = golden("formats_kernels")
    key, idx, vals, dims = next(c for c in cases() if c[0] == case)
    for mode, p in mode_blocks(key):
        mo = tuple(int(x) for x in g[f"{p}/mode_order"])
        assert mo == P.allmode_order(dims, mode)
        tree = P.csf_tree(idx, vals, dims, mo)
        _tree_eq(tree, g, f"{p}/csf", len(dims))
        assert np.array_equal(tree["leaf"], g[f"{p}/csf/leaf"])
        assert np.array_equal(tree["values"], g[f"{p}/csf/values"])
        assert np.array_equal(P.slice_labels(tree), g[f"{p}/labels"])
        h = P.hbcsf(idx, vals, dims, mo)
        assert np.array_equal(h["coo"][0], g[f"{p}/hb/coo/indices"])
        assert np.array_equal(h["coo"][1], g[f"{p}/hb/coo/values"])
        for k in ("slice_ptr", "slice_idx", "rest_idx", "values"):
            assert np.array_equal(h["csl"][k], g[f"{p}/hb/csl/{k}"]), k
        _tree_eq(h["csf"], g, f"{p}/hb/csf", len(dims))
        for _, q, (tau, bs, _ws) in cfg_blocks(p):
            hs = P.split_hbcsf(h, tau)
            assert (hs["csf"] is h["csf"]) == bool(g[f"{q}/split_is_noop"])
            _tree_eq(hs["csf"], g, f"{q}/split", len(dims))
            units, mult = P.block_schedule(hs["csf"], bs)
            assert np.array_equal(units, g[f"{q}/units"])
            assert np.array_equal(mult, g[f"{q}/mult"])
            cs = P.split_tree(tree, tau)
            assert np.array_equal(cs["ptrs"][-1], g[f"{q}/csfsplit/ptr{len(dims) - 2}"])
            fu, _ = P.block_schedule(cs, bs)
            assert np.array_equal(fu, g[f"{q}/csfsplit/units"])


@pytest.mark.parametrize("case", [c[0] for c in cases()])
def test_oracle_mttkrp_matches_reference(case):
    g = golden("formats_kernels")
    key, idx, vals, dims = next(c for c in cases() if c[0] == case)
    for mode, p in mode_blocks(key):
        mo = tuple(int(x) for x in g[f"{p}/mode_order"])
        h = P.hbcsf(idx, vals, dims, mo)
        tree = P.csf_tree(idx, vals, dims, mo)
        for _, q, (tau, bs, _ws) in cfg_blocks(p):
            hs = P.split_hbcsf(h, tau)
            units, _ = P.block_schedule(hs["csf"], bs)
            cs = P.split_tree(tree, tau)
            fu, _ = P.block_schedule(cs, bs)
            for r, fr in rank_blocks(q):
                f = golden_factors(fr, dims, r)
                ref = g[f"{fr}/y"]
                y, ops = P.mttkrp_hbcsf(h, f, mode)
                assert row_dev(y, ref) <= 1e-12
                assert list(ops) == g[f"{fr}/ops_hbcsf"].tolist()
                y, ops = P.mttkrp_hbcsf(hs, f, mode, units=units)
                assert row_dev(y, ref) <= 1e-12
                assert list(ops) == g[f"{fr}/ops_hbsched"].tolist()
                y, ops = P.mttkrp_csf(tree, f, mode)
                assert row_dev(y, ref) <= 1e-12
                assert list(ops) == g[f"{fr}/ops_csf"].tolist()
                y, ops = P.mttkrp_scheduled(cs, fu, f, mode)
                assert row_dev(y, ref) <= 1e-12
                assert list(ops) == g[f"{fr}/ops_sched"].tolist()
                y, ops = P.mttkrp_coo(idx, vals, dims, f, mode)
                assert row_dev(y, ref) <= 1e-12
                assert list(ops) == g[f"{fr}/ops_coo"].tolist()
                if len(vals) <= 400:
                    assert row_dev(loops.mttkrp_entries(idx, vals, dims, f, mode), ref) <= 1e-12


def test_oracle_threads_match_sequential():
    g = golden("formats_kernels")
    key, idx, vals, dims = next(c for c in cases() if c[0] == "skew")
    f = golden_factors("threads", dims, 8)
    for mode in range(3):
        mo = P.allmode_order(dims, mode)
        h = P.split_hbcsf(P.hbcsf(idx, vals, dims, mo), 16)
        units, _ = P.block_schedule(h["csf"], 64)
        y1, k1 = P.mttkrp_hbcsf(h, f, mode, units=units, threads=1)
        y4, k4 = P.mttkrp_hbcsf(h, f, mode, units=units, threads=4)
        assert row_dev(y4, y1) <= 1e-12 and k1 == k4


def test_oracle_canonicalize_bitwise():
    g = golden("canonicalize")
    for key in ("dup_small", "dup_runs", "longrun"):
        idx, vals = P.canonical(g[f"{key}/in_indices"], g[f"{key}/in_values"])
        assert np.array_equal(idx, g[f"{key}/out_indices"])
        assert idx.dtype == np.uint32
        assert vals.tobytes() == g[f"{key}/out_values"].tobytes()
        em = loops.entry_map(g[f"{key}/in_indices"], g[f"{key}/in_values"])
        assert len(em) == len(vals)


def test_oracle_config1_hashes_and_output():
    g = golden("config1")
    idx, vals, dims = g["indices"], g["values"], tuple(int(d) for d in g["dims"])
    mo = P.allmode_order(dims, 0)
    h = P.hbcsf(idx, vals, dims, mo)
    hs = P.split_hbcsf(h, 128)
    units, mult = P.block_schedule(hs["csf"], 512)
    arrays = {
        "coo/indices": h["coo"][0], "coo/values": h["coo"][1],
        "csl/slice_ptr": h["csl"]["slice_ptr"], "csl/slice_idx": h["csl"]["slice_idx"],
        "csl/rest_idx": h["csl"]["rest_idx"], "csl/values": h["csl"]["values"],
        "csf/ptr0": h["csf"]["ptrs"][0], "csf/ptr1": h["csf"]["ptrs"][1],
        "csf/idx0": h["csf"]["idxs"][0], "csf/idx1": h["csf"]["idxs"][1],
        "csf/leaf": h["csf"]["leaf"], "csf/values": h["csf"]["values"],
        "split/ptr0": hs["csf"]["ptrs"][0], "split/ptr1": hs["csf"]["ptrs"][1],
        "split/idx1": hs["csf"]["idxs"][1], "mult": mult, "units": units,
    }
    for name, arr in arrays.items():
        assert digest(arr) == str(g[f"sha/{name}"]), name
    frng = np.random.default_rng(0)
    f = [frng.random((d, 32)).astype(np.float32).astype(np.float64) for d in dims]
    y, ops = P.mttkrp_hbcsf(hs, f, 0)
    assert row_dev(y, g["y"]) <= 1e-12
    assert list(ops) == g["ops"].tolist()
    _, ops2 = P.mttkrp_hbcsf(hs, f, 0, units=units)
    assert list(ops2) == g["ops_sched"].tolist()


def test_oracle_cp_als_fits():
    g = golden("cp_als")
    fits, _, lam = P.cp_als(g["rand/indices"], g["rand/values"], (30, 25, 20), rank=8,
                            max_iters=10, fit_tol=1e-13, seed=2)
    assert np.allclose(fits, g["rand/fits"], atol=1e-10, rtol=0)
    assert np.allclose(lam, g["rand/lam"], rtol=1e-8)
    fits, _, _ = P.cp_als(g["rank2/indices"], g["rank2/values"], (10, 12, 14), rank=2,
                          max_iters=12, fit_tol=1e-13, seed=5)
    assert np.allclose(fits, g["rank2/fits_hbcsf"], atol=1e-10, rtol=0)


# reference known-answer tests (test_formats.py:42-50, test_balance.py:36-152)
def test_oracle_fig_walkthrough():
    from helpers import fig_arrays

    idx, vals = fig_arrays()
    t = P.csf_tree(idx, vals, (3, 3, 4), (0, 1, 2))
    assert t["idxs"][0].tolist() == [0, 1, 2]
    assert t["ptrs"][0].tolist() == [0, 1, 4, 5]
    assert t["idxs"][1].tolist() == [0, 0, 1, 2, 1]
    assert t["ptrs"][1].tolist() == [0, 1, 2, 3, 4, 8]
    assert t["leaf"].tolist() == [0, 0, 1, 2, 0, 1, 2, 3]
    assert P.slice_labels(t).tolist() == [0, 1, 2]
    h = P.hbcsf(idx, vals, (3, 3, 4), (0, 1, 2))
    assert h["csl"]["slice_idx"].tolist() == [1] and h["csl"]["values"].tolist() == [2.0, 3.0, 4.0]


def _line(n):
    idx = np.stack([np.zeros(n, np.int64), np.zeros(n, np.int64), np.arange(n)], axis=1)
    return idx.astype(np.uint32), np.arange(1.0, n + 1.0)


def test_oracle_split_and_schedule_kats():
    idx, vals = _line(32)
    t = P.split_tree(P.csf_tree(idx, vals, (1, 1, 32), (0, 1, 2)), 16)
    assert np.diff(t["ptrs"][-1]).tolist() == [16, 16] and t["idxs"][1].tolist() == [0, 0]
    idx, vals = _line(33)
    t = P.split_tree(P.csf_tree(idx, vals, (1, 1, 33), (0, 1, 2)), 16)
    assert np.diff(t["ptrs"][-1]).tolist() == [16, 16, 1]
    idx, vals = _line(2048)
    t = P.split_tree(P.csf_tree(idx, vals, (1, 1, 2048), (0, 1, 2)), 128)
    units, mult = P.block_schedule(t, 512)
    assert mult.tolist() == [4] and len(units) == 4
    idx = np.stack([np.zeros(32, np.int64), np.repeat(np.arange(8), 4), np.tile(np.arange(4), 8)], axis=1)
    t = P.csf_tree(idx.astype(np.uint32), np.ones(32), (1, 8, 4), (0, 1, 2))
    units, mult = P.block_schedule(t, 16)
    assert mult.tolist() == [2]
    sizes = np.diff(t["ptrs"][-1])
    assert [int(sizes[u[2]:u[3]].sum()) for u in units] == [16, 16]
