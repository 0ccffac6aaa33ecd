"""Randomised sweep in the shape of the reference's acceptance criteria 04/05
(test_acceptance.py:136-189): many small tensors of order 3 and 4, ranks
1/8/32 (and 12 / 48 for the float4 passes), every kernel variant — COO, CSF,
split CSF (B-CSF), HB-CSF, split HB-CSF, scheduled — against the
entry-at-a-time loop oracle, with SplitConfig(4, 8, 2) so fibers and slices
actually split; split invariance of the device result (criterion 05)."""
from __future__ import annotations

import numpy as np
import pytest

from helpers import row_dev
from oracle import loops

pytestmark = pytest.mark.gpu

TOL = 1e-4


def _instance(rng, order):
    dims = tuple(int(d) for d in rng.integers(2, 9, order))
    cap = int(np.prod(dims))
    nnz = int(rng.integers(1, min(cap, 260) + 1))
    flats = rng.choice(cap, size=nnz, replace=False)
    if rng.random() < 0.5:  # concentrate entries on a few slices: heavy, split slices
        hot = rng.choice(cap, size=max(1, nnz // 8), replace=False)
        flats = np.unique(np.concatenate([flats[: nnz // 2], hot]))
    idx = np.empty((len(flats), order), dtype=np.int64)
    rem = flats.copy()
    for d in range(order - 1, -1, -1):
        idx[:, d] = rem % dims[d]
        rem //= dims[d]
    return dims, idx.astype(np.uint32), rng.uniform(0.1, 1.0, len(flats))


@pytest.mark.parametrize("block", range(5))
def test_random_instances_all_kernels(block):
    import paper_1904_03329_b200 as hb

    rng = np.random.default_rng(20240817 + block)
    cfg = hb.SplitConfig(4, 8, 2)
    ranks = (1, 8, 32, 12, 48)
    for inst in range(20):  # 5 blocks x 20 = 100 instances
        order = 3 if inst % 2 == 0 else 4
        rank = ranks[(inst // 2 + block) % len(ranks)]
        dims, idx, vals = _instance(rng, order)
        t = hb.CooTensor(dims, idx, vals)
        f = [rng.standard_normal((d, rank)).astype(np.float32).astype(np.float64) for d in dims]
        for mode in range(order):
            ref = loops.mttkrp_entries(idx, vals, dims, f, mode)
            mo = hb.allmode_order(dims, mode)
            c = hb.build_csf(t, mo)
            cs = hb.split_fibers(c, cfg)
            h = hb.build_hbcsf(t, mo)
            hs = hb.split_fibers(h, cfg)
            sched = hb.assign_slice_blocks(hs.csf_part, cfg)
            outs = {
                "coo": hb.mttkrp(t, f, mode)[0],
                "csf": hb.mttkrp(c, f, mode)[0],
                "bcsf": hb.mttkrp(cs, f, mode)[0],
                "hbcsf": hb.mttkrp(h, f, mode)[0],
                "hbcsf_split": hb.mttkrp(hs, f, mode)[0],
                "scheduled": hb.mttkrp_hbcsf(hs, f, mode, schedule=sched)[0],
            }
            for name, y in outs.items():
                dev = row_dev(y, ref)
                assert dev <= TOL, (block, inst, dims, rank, mode, name, dev)
            # criterion 05: splitting does not change the device result beyond
            # fp32 reassociation
            assert row_dev(outs["hbcsf_split"], outs["hbcsf"]) <= 1e-5
