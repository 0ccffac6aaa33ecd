"""Plan-internal mode order: MTTKRP time per mode with the reference order
(allmode_order: rest by ascending dim) vs the swapped order of the two
non-target modes.  Same output (the sum over nonzeros does not depend on the
tree order); the question is which factor is gathered per nonzero (leaf) and
which per fiber, and how many fibers there are."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

import paper_1904_03329_b200 as hb
from paper_1904_03329_b200.generate import CONFIGS, config_tensor
from paper_1904_03329_b200.kernels import mttkrp_device

cfgs = sys.argv[1:] or ["nell-2"]


def timed(fn, n=10):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n


for cfg in cfgs:
    dims = CONFIGS[cfg]["dims"]
    t = config_tensor(cfg)
    f = [torch.rand((d, 32), device="cuda") for d in dims]
    sc = hb.SplitConfig()
    for mode in range(3):
        mo = hb.allmode_order(dims, mode)
        res = []
        ys = []
        for order in (mo, (mo[0], mo[2], mo[1])):
            h = hb.split_fibers(hb.build_hbcsf(t, order), sc)
            nf = h.csf_part.num_fibers if h.csf_part.nnz else 0
            y, _ = mttkrp_device(h, f, mode)
            ys.append(y.clone())
            ms = timed(lambda: mttkrp_device(h, f, mode, out=y))
            res.append((order, ms, nf, h.csf_part.nnz, h.csl_part.nnz, h.coo_part.nnz))
            del h
            torch.cuda.empty_cache()
        d = ((ys[0] - ys[1]).norm(dim=1) / (1 + ys[0].norm(dim=1))).max().item()
        for order, ms, nf, m_csf, m_csl, m_coo in res:
            print(f"{cfg} mode {mode} order {order}: {ms:.3f} ms  csf nnz {m_csf} fibers {nf} "
                  f"csl {m_csl} coo {m_coo}", flush=True)
        print(f"{cfg} mode {mode}: row dev between orders {d:.2e}", flush=True)
    del t
    torch.cuda.empty_cache()
