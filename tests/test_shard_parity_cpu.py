"""The premise of the at-scale parity check (oracle/shard_parity.py), on the
CPU: the reference algorithm's arrays for a whole tensor, restricted to a set
of slices, equal its arrays for those slices alone — formats, split trees,
schedule units and MTTKRP rows (SURVEY §7 hard part 6)."""
import numpy as np
import pytest

from oracle import shard_parity as S
from oracle import tenkit_port as P


def _tensor(seed, dims=(60, 40, 80), m=6000):
    rng = np.random.default_rng(seed)
    # skewed first mode: heavy slices (split + multi-unit schedules), many light
    i0 = np.minimum((rng.pareto(1.2, m) * 3).astype(np.int64), dims[0] - 1)
    idx = np.stack([i0, rng.integers(0, dims[1], m), rng.integers(0, dims[2], m)], 1)
    # singleton slices for the COO bucket, singleton-fiber slices for CSL
    extra = np.array([[dims[0] - 1, 1, 2], [dims[0] - 2, 3, 4], [dims[0] - 2, 5, 6], [dims[0] - 3, 7, 8]])
    return P.canonical(np.vstack([idx, extra]).astype(np.uint32), rng.random(m + 4) + 0.1)


@pytest.mark.parametrize("mode", [0, 1, 2])
def test_restricted_full_build_equals_shard_build(mode):
    dims = (60, 40, 80)
    idx, val = _tensor(7 + mode, dims)
    mo = P.allmode_order(dims, mode)
    full = P.hbcsf(idx, val, dims, mo)
    fs = P.split_hbcsf(full, 8)
    units, mult = P.block_schedule(fs["csf"], 64)
    hist = np.bincount(idx[:, mode], minlength=dims[mode])
    rows = S.select_slices(hist, 1500, seed=mode, runs=2, run_len=5)
    assert len(rows) > 3
    si, sv, h, hs, su, sm = S.oracle_shard(idx, val, dims, mode, rows, tau=8, block_size=64)
    gpu_like = {"coo": full["coo"], "csl": full["csl"], "csf": dict(fs["csf"]),
                "labels": (P.csf_tree(idx, val, dims, mo)["idxs"][0], full["labels"])}
    gpu_like["csf"]["leaf"] = fs["csf"]["leaf"]
    res = S.compare_hbcsf(gpu_like, hs, rows)
    assert all(res.values()), res
    _, _, _, _, pos = S.restrict_tree(fs["csf"]["ptrs"], fs["csf"]["idxs"], fs["csf"]["leaf"],
                                      fs["csf"]["values"], rows)
    ru, rm = S.restrict_units(units, mult, fs["csf"]["ptrs"][0], pos)
    assert np.array_equal(ru, su)
    assert np.array_equal(rm, sm)
    f = [np.random.default_rng(3).random((d, 8)) for d in dims]
    y_full, _ = P.mttkrp_hbcsf(fs, f, mode)
    y_shard, ops = P.mttkrp_hbcsf(hs, f, mode)
    assert np.allclose(y_full[rows], y_shard[rows], rtol=1e-12, atol=0)
    c = hs["csl"]
    ls = [len(x) for x in hs["csf"]["idxs"]]
    assert S.opcount_formula(len(hs["coo"][1]), len(c["values"]), ls, len(hs["csf"]["values"]), 3, 8) == ops
    _, ops_s = P.mttkrp_hbcsf(hs, f, mode, units=su)
    assert S.opcount_formula(len(hs["coo"][1]), len(c["values"]), ls, len(hs["csf"]["values"]), 3, 8,
                             units=len(su)) == ops_s


def test_stratified_sample_caps_heavy_slices():
    hist = np.array([5000, 10, 0, 300, 7, 1, 1, 40, 2, 900] * 20)
    rows = S.stratified_slices(hist, 2000, seed=1, max_slice_frac=0.25)
    assert hist[rows].max() <= 500
    assert 0 < hist[rows].sum() < 6000
