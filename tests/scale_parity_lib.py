"""Runner of the at-scale oracle parity check (oracle/shard_parity.py) on the
GPU: the full benchmark tensor is generated and built on the device
(libhbk: K1 wide-key sort, K2-K3 HB-CSF, K4 split, K5 schedule, K6-K8
MTTKRP); the oracle (oracle/tenkit_port.py, the restated reference) sees only
a whole-slice shard of it.  Used by tests/test_gpu_scale_parity.py (bounded
shards) and scripts/scale_parity.py (>= 10M-nonzero shards, evidence under
profiles/)."""
from __future__ import annotations

import time

import numpy as np

from oracle import shard_parity as S
from oracle import tenkit_port as P

RANK = 32


def make_factors(dims, seed, rank=RANK):
    rng = np.random.default_rng(seed)  # cli.py:274-276 convention
    return [rng.random((d, rank)) for d in dims]


def run_config(config: str, target_nnz: int, modes=None, seed: int = 0, log=print) -> list[dict]:
    import torch

    import paper_1904_03329_b200 as hb
    from paper_1904_03329_b200.generate import CONFIGS, config_tensor
    from paper_1904_03329_b200.kernels import mttkrp_device

    cfg = CONFIGS[config]
    dims = tuple(cfg["dims"])
    tic = time.perf_counter()
    t = config_tensor(config)
    idx, val = t.indices, t.values
    log(f"[{config}] generated {t.nnz} nnz, exported ({time.perf_counter() - tic:.1f}s)")
    f64 = make_factors(dims, cfg["seed"])
    f32 = [torch.from_numpy(f).float().cuda() for f in f64]
    f64r = [f.float().double().cpu().numpy() for f in f32]  # what the fp32 kernel sees
    split = hb.SplitConfig()
    out = []
    for mode in (range(len(dims)) if modes is None else modes):
        rec = {"config": config, "mode": mode, "nnz": t.nnz}
        tic = time.perf_counter()
        mo = hb.allmode_order(dims, mode)
        full = hb.build_csf(t, mo)
        labels = (full.idxs[0].copy(), hb.classify_slices(full))
        del full
        h = hb.split_fibers(hb.build_hbcsf(t, mo), split)
        sched = hb.assign_slice_blocks(h.csf_part, split)
        y, ops = mttkrp_device(h, f32, mode)
        ys, ops_s = mttkrp_device(h, f32, mode, schedule=sched)
        torch.cuda.synchronize()
        gpu = S.gpu_arrays(h, labels)
        units, mult = sched.units_array(), sched.multiplicities
        rec["gpu_s"] = time.perf_counter() - tic

        hist = np.bincount(idx[:, mode], minlength=dims[mode])
        rows = S.select_slices(hist, target_nnz, seed=seed + mode)
        tic = time.perf_counter()
        si, sv, h_o, hs_o, units_o, mult_o = S.oracle_shard(idx, val, dims, mode, rows)
        rec.update(shard_slices=int(len(rows)), shard_nnz=int(len(sv)),
                   heaviest_slice_nnz=int(hist.max()),
                   shard_census={"coo": int(len(hs_o["coo"][1])),
                                 "csl_slices": int(len(hs_o["csl"]["slice_idx"])),
                                 "csl": int(len(hs_o["csl"]["values"])),
                                 "csf_slices": int(len(hs_o["csf"]["idxs"][0])),
                                 "csf": int(len(hs_o["csf"]["values"]))})
        arrays = S.compare_hbcsf(gpu, hs_o, rows)
        _, _, _, _, pos = S.restrict_tree(gpu["csf"]["ptrs"], gpu["csf"]["idxs"], gpu["csf"]["leaf"],
                                          gpu["csf"]["values"], rows)
        ru, rm = S.restrict_units(units, mult, gpu["csf"]["ptrs"][0], pos)
        arrays["schedule_units"] = bool(np.array_equal(ru, units_o))
        arrays["schedule_multiplicities"] = bool(np.array_equal(rm, mult_o))
        rec["arrays_bit_exact"] = {k: bool(v) for k, v in arrays.items()}
        rec["bit_exact"] = all(arrays.values())

        y_o, ops_o = P.mttkrp_hbcsf(hs_o, f64r, mode)
        rows_gpu = y[torch.from_numpy(rows).cuda()].double().cpu().numpy()
        rows_gpu_s = ys[torch.from_numpy(rows).cuda()].double().cpu().numpy()
        rec["max_row_dev"] = P.row_deviation(rows_gpu, y_o[rows])
        rec["max_row_dev_scheduled"] = P.row_deviation(rows_gpu_s, y_o[rows])
        # OpCount: the structure formula reproduces the oracle's counts on the
        # shard, and libhbk's full-size counts from the full-size structure
        c = hs_o["csl"]
        ls_o = [len(x) for x in hs_o["csf"]["idxs"]]
        f_shard = S.opcount_formula(len(hs_o["coo"][1]), len(c["values"]), ls_o,
                                    len(hs_o["csf"]["values"]), len(dims), RANK)
        ls = list(h.csf_part.level_sizes())
        f_full = S.opcount_formula(h.coo_part.nnz, h.csl_part.nnz, ls, h.csf_part.nnz, len(dims), RANK)
        f_full_s = S.opcount_formula(h.coo_part.nnz, h.csl_part.nnz, ls, h.csf_part.nnz, len(dims), RANK,
                                     units=len(units))
        rec["opcount_exact"] = bool(tuple(f_shard) == tuple(ops_o)
                                    and tuple(f_full) == (ops.muls, ops.adds)
                                    and tuple(f_full_s) == (ops_s.muls, ops_s.adds))
        rec["oracle_s"] = time.perf_counter() - tic
        log(f"[{config}] mode {mode}: shard {rec['shard_nnz']} nnz / {rec['shard_slices']} slices, "
            f"bit_exact={rec['bit_exact']} row_dev={rec['max_row_dev']:.2e}/"
            f"{rec['max_row_dev_scheduled']:.2e} opcount={rec['opcount_exact']} "
            f"(gpu {rec['gpu_s']:.1f}s, oracle {rec['oracle_s']:.1f}s)")
        if not rec["bit_exact"]:
            log(f"   mismatching arrays: {[k for k, v in arrays.items() if not v]}")
        out.append(rec)
        del h, sched, y, ys, gpu
        torch.cuda.empty_cache()
    return out
