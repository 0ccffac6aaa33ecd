"""Maximum-extent cases: mode lengths past the kernels' index-width limits
(2^27: pre-scaled B-position streams; 2^29: the fast path's flag bits), so
the R = 32 plan falls back to the runtime-stride kernels and the fast path to
the generic kernel.  The factors are tens of GB, so they live on the device;
the check gathers only the rows the nonzeros touch (float64 of the fp32
values) and compares against a NumPy sum over the entries (kernels.py:109-151
semantics), plus zero rows everywhere else."""
from __future__ import annotations

import numpy as np
import pytest

from helpers import row_dev

pytestmark = pytest.mark.gpu


def _entries_mttkrp(torch, idx, vals, f, mode):
    """(touched output rows, their rows) from the touched factor rows only."""
    rows, inv = np.unique(idx[:, mode], return_inverse=True)
    prod = np.repeat(vals[:, None], f[(mode + 1) % 3].shape[1], 1)
    for d in range(3):
        if d == mode:
            continue
        sel = torch.from_numpy(idx[:, d].astype(np.int64)).cuda()
        prod = prod * f[d].index_select(0, sel).double().cpu().numpy()
    y = np.zeros((len(rows), prod.shape[1]))
    np.add.at(y, inv, prod)
    return rows, y


@pytest.mark.parametrize("big,rank", [((1 << 27) + 3, 32), ((1 << 29) + 1, 4)])
def test_large_extent(big, rank):
    import torch

    import paper_1904_03329_b200 as hb
    from paper_1904_03329_b200.kernels import plan_for

    free, _ = torch.cuda.mem_get_info()
    need = 2 * big * rank * 4 + (4 << 30)
    if free < need:
        pytest.skip(f"needs {need >> 30} GB of free device memory")
    rng = np.random.default_rng(11)
    dims = (50, 40, big)
    nnz = 20000
    idx = np.stack([rng.integers(0, 50, nnz), rng.integers(0, 40, nnz),
                    np.concatenate([rng.integers(0, big, nnz - 4), [0, 1, big - 2, big - 1]])],
                   1).astype(np.uint32)
    idx = np.unique(idx, axis=0)
    vals = rng.uniform(0.1, 1.0, len(idx))
    t = hb.CooTensor(dims, idx, vals)
    f = [torch.rand((d, rank), device="cuda") for d in dims]
    for mode in range(3):
        h = hb.build_hbcsf(t, hb.allmode_order(dims, mode))
        y, _ = hb.mttkrp_device(h, f, mode)
        # leaf / fiber extents >= 2^29 leave the float4 kernels for the generic one
        wide = big >= (1 << 29) and mode != 2
        assert plan_for(h, mode, rank).info.fast_path == (0 if wide else 1)
        rows, ref = _entries_mttkrp(torch, idx, vals, f, mode)
        sel = torch.from_numpy(rows.astype(np.int64)).cuda()
        assert row_dev(y.index_select(0, sel).double().cpu().numpy(), ref) <= 1e-4
        # every other row is zero
        y.index_fill_(0, sel, 0.0)
        assert int(torch.count_nonzero(y)) == 0
        del y
    del f
    torch.cuda.empty_cache()
