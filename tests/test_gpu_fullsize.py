"""Parity at benchmark scale through size-independent properties (the CPU
oracle is too slow here): on the Appendix-A generator's tensors, the fast
fp32 kernels (B-position streams, padded heavy layout, CSL/COO/zero tasks)
against libhbk's independent generic kernel run in fp64 (HBK_F64_GENERIC) —
different code, different layout, different arithmetic — with the
reference's row metric; the fp64 fast path against the same generic kernel;
plus linearity in a factor and bit-repeatability of the fast path."""
from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _rowdev(y, ref):
    import torch

    num = torch.linalg.vector_norm(y.double() - ref, dim=1)
    return float((num / (1.0 + torch.linalg.vector_norm(ref, dim=1))).max())


@pytest.mark.parametrize("config,scale", [("nell-2", 1.0), ("flickr-3d", 0.5),
                                          ("delicious-3d", 0.5), ("nell-1", 0.5)])
def test_fast_fp32_matches_generic_fp64_at_scale(config, scale, monkeypatch):
    import torch

    import paper_1904_03329_b200 as hb
    from paper_1904_03329_b200.generate import CONFIGS, config_tensor
    from paper_1904_03329_b200.kernels import mttkrp_device

    dims = CONFIGS[config]["dims"]
    t = config_tensor(config, scale=scale)
    g = torch.Generator(device="cuda").manual_seed(7)
    f64 = [torch.rand((d, 32), dtype=torch.float64, device="cuda", generator=g) for d in dims]
    f32 = [f.float() for f in f64]
    f64r = [f.double() for f in f32]  # the fp64 kernel sees the fp32-rounded factors
    for mode in range(3):
        h = hb.split_fibers(hb.build_hbcsf(t, hb.allmode_order(dims, mode)), hb.SplitConfig())
        y32, _ = mttkrp_device(h, f32, mode)
        monkeypatch.setenv("HBK_F64_GENERIC", "1")  # the independent generic fp64 kernel
        y64, _ = mttkrp_device(h, f64r, mode)
        monkeypatch.delenv("HBK_F64_GENERIC")
        assert y32.dtype == torch.float32 and y64.dtype == torch.float64
        assert _rowdev(y32, y64) <= 1e-4, (config, mode)
        # the fp64 fast path (same streams and tasks as fp32, double2 lanes,
        # fp64 value streams) against the generic fp64 kernel
        h2 = hb.split_fibers(hb.build_hbcsf(t, hb.allmode_order(dims, mode)), hb.SplitConfig())
        y64f, _ = mttkrp_device(h2, f64r, mode)
        assert _rowdev(y64f, y64) <= 1e-12, (config, mode)
        del h2
        # linearity in a factor: Y(2C) = 2 Y(C) exactly, except that the
        # chunks of a split slice (thousands for the 3M-nonzero nell-2 slices)
        # meet in red.global.add order, which varies run to run: fp32
        # reassociation, ~1e-6 of the row norm (a bug would show as O(1))
        fs = list(f32)
        d = hb.allmode_order(dims, mode)[2]
        fs[d] = f32[d] * 2.0
        y2, _ = mttkrp_device(h, fs, mode)
        assert _rowdev(y2, 2.0 * y32.double()) <= 1e-5
        # repeatability up to the same atomic order
        y32b, _ = mttkrp_device(h, f32, mode)
        assert _rowdev(y32b, y32.double()) <= 1e-5


@pytest.mark.parametrize("R", [8, 16, 48, 64])
def test_other_ranks_fast_path_at_scale(R):
    """R a multiple of 4 takes the float4 kernels in passes of 32 columns;
    checked against the generic fp64 kernel on a nell-2-shaped tensor."""
    import torch

    import paper_1904_03329_b200 as hb
    from paper_1904_03329_b200.generate import CONFIGS, config_tensor
    from paper_1904_03329_b200.kernels import mttkrp_device, plan_for

    dims = CONFIGS["nell-2"]["dims"]
    t = config_tensor("nell-2", scale=0.05)
    g = torch.Generator(device="cuda").manual_seed(R)
    f32 = [torch.rand((d, R), device="cuda", generator=g) for d in dims]
    for mode in range(3):
        h = hb.build_hbcsf(t, hb.allmode_order(dims, mode))
        assert plan_for(h, mode, R).info.fast_path == 1
        y32, _ = mttkrp_device(h, f32, mode)
        y64, _ = mttkrp_device(h, [f.double() for f in f32], mode)
        assert _rowdev(y32, y64) <= 1e-4, (R, mode)


@pytest.mark.parametrize("config,scale", [("nell-2", 1.0), ("nell-1", 0.5), ("delicious-3d", 0.5)])
def test_cp_als_fused_matches_fp64_at_scale(config, scale):
    """CP-ALS at benchmark scale: the R = 32 fused fp32 sweep (MTTKRP fast
    path + tensor-core 3xTF32 row update + M^T G_Y M Gram) against the same
    solve with the fp64 MTTKRP and fp64 factors — fits, weights and the
    normalised factors."""
    import paper_1904_03329_b200 as hb
    from paper_1904_03329_b200.generate import config_tensor

    t = config_tensor(config, scale=scale)
    m32, h32 = hb.cp_als(t, rank=32, max_iters=4, fit_tol=0.0, seed=5)
    m64, h64 = hb.cp_als(t, rank=32, max_iters=4, fit_tol=0.0, seed=5, mttkrp_precision="fp64")
    f32, f64 = np.array([h.fit for h in h32]), np.array([h.fit for h in h64])
    assert len(f32) == len(f64) == 5
    # the first record is the random initial model (fit far below 0)
    assert np.allclose(f32[1:], f64[1:], atol=2e-6, rtol=0), (f32, f64)
    assert np.allclose(m32.lam, m64.lam, rtol=2e-3)
    for a, b in zip(m32.factors, m64.factors):
        cos = np.abs((a * b).sum(0)) / (np.linalg.norm(a, axis=0) * np.linalg.norm(b, axis=0))
        assert cos.min() > 0.999
