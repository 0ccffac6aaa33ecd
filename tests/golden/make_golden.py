"""Generate golden fixtures by running the REFERENCE implementation.

Run in the build container, where the read-only reference exists:

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

It imports ``tenkit`` from /root/reference/pkg/src (never copied into the
repo) and records, for a fixed set of seeded inputs, the reference's outputs
of every hot-path function: CSF / HB-CSF arrays, slice labels, fiber-split
arrays, block schedules, MTTKRP outputs and OpCounts, canonicalize results
and CP-ALS fit histories.  Small arrays are stored verbatim; arrays of the
100K-nonzero configuration-1 case are stored as SHA-256 digests of their
exact bytes (int64 pointers / uint32 indices / float64 values).

The fixtures (tests/golden/*.npz) are committed; tests read only them, so
nothing at test time needs /root/reference.
"""
from __future__ import annotations

import hashlib
import zlib
import json
import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent
sys.dont_write_bytecode = True
sys.path.insert(0, str(REF))

import tenkit as tk  # noqa: E402
from tenkit.balance import SplitConfig, assign_slice_blocks, split_fibers  # noqa: E402
from tenkit.kernels import mttkrp_coo, mttkrp_csf, mttkrp_hbcsf, mttkrp_scheduled  # noqa: E402

FIG_TEXT = """\
1 1 1 1.0
2 1 1 2.0
2 2 2 3.0
2 3 3 4.0
3 2 1 5.0
3 2 2 6.0
3 2 3 7.0
3 2 4 8.0
"""


def digest(a: np.ndarray) -> str:
    a = np.ascontiguousarray(a)
    return hashlib.sha256(a.dtype.str.encode() + str(a.shape).encode() + a.tobytes()).hexdigest()


def golden_factors(key: str, dims, rank):
    """Factors of a fixture, regenerated from the key (no need to store them):
    uniform(0,1) rounded through float32 so the GPU sees the same values."""
    rng = np.random.default_rng(zlib.crc32(key.encode()))
    return [rng.random((d, rank)).astype(np.float32).astype(np.float64) for d in dims]


def random_tensor(rng, dims, nnz):
    cap = int(np.prod([np.int64(d) for d in dims]))
    flats = rng.choice(cap, size=nnz, replace=False)
    idx = np.empty((nnz, len(dims)), dtype=np.int64)
    rem = flats
    for d in range(len(dims) - 1, -1, -1):
        idx[:, d] = rem % dims[d]
        rem = rem // dims[d]
    return tk.canonicalize(tk.CooTensor(dims, idx, rng.uniform(0.1, 1.0, size=nnz)))


def record_case(store: dict, key: str, t, cfgs, ranks, rng, big=False):
    """All hot-path outputs of tensor t for every mode."""
    put = (lambda k, a: store.__setitem__(k, np.asarray(digest(np.asarray(a))))) if big else \
        (lambda k, a: store.__setitem__(k, np.asarray(a)))
    if not big:
        store[f"{key}/indices"] = t.indices
        store[f"{key}/values"] = t.values
    store[f"{key}/dims"] = np.asarray(t.dims)
    for mode in range(t.order):
        mo = tk.allmode_order(t.dims, mode)
        p = f"{key}/m{mode}"
        store[f"{p}/mode_order"] = np.asarray(mo)
        c = tk.build_csf(t, mo)
        for d in range(t.order - 1):
            put(f"{p}/csf/ptr{d}", c.ptrs[d])
            put(f"{p}/csf/idx{d}", c.idxs[d])
        put(f"{p}/csf/leaf", c.leaf_idx)
        put(f"{p}/csf/values", c.values)
        put(f"{p}/labels", tk.classify_slices(c))
        h = tk.build_hbcsf(t, mo)
        put(f"{p}/hb/coo/indices", h.coo_part.indices)
        put(f"{p}/hb/coo/values", h.coo_part.values)
        put(f"{p}/hb/csl/slice_ptr", h.csl_part.slice_ptr)
        put(f"{p}/hb/csl/slice_idx", h.csl_part.slice_idx)
        put(f"{p}/hb/csl/rest_idx", h.csl_part.rest_idx)
        put(f"{p}/hb/csl/values", h.csl_part.values)
        for d in range(t.order - 1):
            put(f"{p}/hb/csf/ptr{d}", h.csf_part.ptrs[d])
            put(f"{p}/hb/csf/idx{d}", h.csf_part.idxs[d])
        put(f"{p}/hb/csf/leaf", h.csf_part.leaf_idx)
        put(f"{p}/hb/csf/values", h.csf_part.values)
        for ci, cfg in enumerate(cfgs):
            q = f"{p}/cfg{ci}"
            store[f"{q}/cfg"] = np.asarray([cfg.fiber_threshold, cfg.block_size, cfg.warp_size])
            hs = split_fibers(h, cfg)
            store[f"{q}/split_is_noop"] = np.asarray(hs.csf_part is h.csf_part)
            for d in range(t.order - 1):
                put(f"{q}/split/ptr{d}", hs.csf_part.ptrs[d])
                put(f"{q}/split/idx{d}", hs.csf_part.idxs[d])
            sched = assign_slice_blocks(hs.csf_part, cfg)
            units = np.array([[u.block_id, u.slice_pos, u.fiber_start, u.fiber_stop]
                              for u in sched.units], dtype=np.int64).reshape(-1, 4)
            put(f"{q}/units", units)
            put(f"{q}/mult", sched.multiplicities)
            cs = split_fibers(c, cfg)
            put(f"{q}/csfsplit/ptr{t.order - 2}", cs.ptrs[t.order - 2])
            full_sched = assign_slice_blocks(cs, cfg)
            fu = np.array([[u.block_id, u.slice_pos, u.fiber_start, u.fiber_stop]
                           for u in full_sched.units], dtype=np.int64).reshape(-1, 4)
            put(f"{q}/csfsplit/units", fu)
            for r in ranks:
                fr = f"{q}/r{r}"
                ff = golden_factors(fr, t.dims, r)
                # every variant computes the same MTTKRP; the reference's own
                # outputs agree to 1e-10 (test_acceptance.py:136-166), so one
                # output is stored and all variants are checked against it
                y, ops = mttkrp_hbcsf(h, ff, mode)
                store[f"{fr}/y"] = y
                store[f"{fr}/ops_hbcsf"] = np.asarray([ops.muls, ops.adds])
                for name, (yy, oo) in {
                    "hbsched": mttkrp_hbcsf(hs, ff, mode, schedule=sched),
                    "csf": mttkrp_csf(c, ff, mode),
                    "sched": mttkrp_scheduled(cs, full_sched, ff, mode),
                    "coo": mttkrp_coo(t, ff, mode),
                }.items():
                    assert float(np.max(np.abs(yy - y), initial=0.0)) <= 1e-9 * (1 + np.abs(y).max(initial=0))
                    store[f"{fr}/ops_{name}"] = np.asarray([oo.muls, oo.adds])


def main():
    # -- formats/balance/kernels on small tensors --------------------------
    small = {}
    fig = tk.canonicalize(tk.parse_frostt(FIG_TEXT))
    record_case(small, "fig", fig, [SplitConfig(2, 2, 1), SplitConfig()], [1, 4, 32],
                np.random.default_rng(1))
    rng = np.random.default_rng(20240817)
    cases = [
        ("r3a", (9, 7, 6), 120), ("r3b", (40, 8, 8), 300), ("r3c", (30, 6, 6), 120),
        ("r3d", (12, 8, 25), 380), ("r3e", (25, 12, 12), 140),
        ("r4a", (6, 5, 4, 3), 90), ("r4b", (12, 6, 5, 4), 220), ("r4c", (7, 6, 5, 4), 150),
    ]
    for key, dims, nnz in cases:
        t = random_tensor(rng, dims, nnz)
        record_case(small, key, t, [SplitConfig(4, 8, 2), SplitConfig(16, 64, 32)], [1, 8, 32], rng)
    # skewed tensor from the reference generator: heavy slices, long fibers
    sk = tk.generate_tensor((40, 300, 200), 20000, skew=1.5, seed=3)
    record_case(small, "skew", sk, [SplitConfig(16, 64, 32), SplitConfig()], [32], rng)
    np.savez_compressed(OUT / "formats_kernels.npz", **small)

    # -- canonicalize with duplicate runs and cancellations ---------------
    can = {}
    crng = np.random.default_rng(7)
    for key, n, span in (("dup_small", 400, 6), ("dup_runs", 3000, 3)):
        idx = crng.integers(0, span, size=(n, 3))
        vals = crng.standard_normal(n) * 10 ** crng.uniform(-3, 3, n)
        # exact cancellations: pairs (+x, -x) on fresh coordinates
        extra = crng.integers(span, span + 4, size=(20, 3))
        x = crng.random(20)
        idx = np.vstack([idx, extra, extra])
        vals = np.concatenate([vals, x, -x])
        t = tk.CooTensor((span + 4,) * 3, idx, vals)
        c = tk.canonicalize(t)
        can[f"{key}/in_indices"] = t.indices
        can[f"{key}/in_values"] = t.values
        can[f"{key}/out_indices"] = c.indices
        can[f"{key}/out_values"] = c.values
    # one long run (> 128 duplicates) to exercise the pairwise recursion
    idx = np.zeros((700, 3), dtype=np.int64)
    vals = crng.standard_normal(700) * 10 ** crng.uniform(-4, 4, 700)
    t = tk.CooTensor((2, 2, 2), idx, vals)
    c = tk.canonicalize(t)
    can["longrun/in_indices"], can["longrun/in_values"] = t.indices, t.values
    can["longrun/out_indices"], can["longrun/out_values"] = c.indices, c.values
    np.savez_compressed(OUT / "canonicalize.npz", **can)

    # -- configuration 1 (BASELINE.json configs[0]) -----------------------
    c1 = {}
    t1 = tk.generate_tensor((1000, 1000, 1000), 100_000, skew=0.0, seed=0)
    c1["indices"] = t1.indices
    c1["values"] = t1.values
    c1["dims"] = np.asarray(t1.dims)
    mo = tk.allmode_order(t1.dims, 0)
    cfg = SplitConfig()
    h = tk.build_hbcsf(t1, mo)
    hs = split_fibers(h, cfg)
    sched = assign_slice_blocks(hs.csf_part, cfg)
    for name, arr in [("coo/indices", h.coo_part.indices), ("coo/values", h.coo_part.values),
                      ("csl/slice_ptr", h.csl_part.slice_ptr), ("csl/slice_idx", h.csl_part.slice_idx),
                      ("csl/rest_idx", h.csl_part.rest_idx), ("csl/values", h.csl_part.values),
                      ("csf/ptr0", h.csf_part.ptrs[0]), ("csf/ptr1", h.csf_part.ptrs[1]),
                      ("csf/idx0", h.csf_part.idxs[0]), ("csf/idx1", h.csf_part.idxs[1]),
                      ("csf/leaf", h.csf_part.leaf_idx), ("csf/values", h.csf_part.values),
                      ("split/ptr0", hs.csf_part.ptrs[0]), ("split/ptr1", hs.csf_part.ptrs[1]),
                      ("split/idx1", hs.csf_part.idxs[1]), ("mult", sched.multiplicities)]:
        c1[f"sha/{name}"] = np.asarray(digest(np.asarray(arr)))
    units = np.array([[u.block_id, u.slice_pos, u.fiber_start, u.fiber_stop] for u in sched.units],
                     dtype=np.int64).reshape(-1, 4)
    c1["sha/units"] = np.asarray(digest(units))
    c1["census"] = np.asarray([h.coo_part.nnz, h.csl_part.num_slices, h.csf_part.num_slices,
                               h.csl_part.nnz, h.csf_part.nnz, h.csf_part.num_fibers])
    frng = np.random.default_rng(0)  # cli.py:274-276 convention, seed 0
    f = [frng.random((d, 32)).astype(np.float32).astype(np.float64) for d in t1.dims]
    y, ops = mttkrp_hbcsf(hs, f, 0)
    c1["y"] = y
    c1["ops"] = np.asarray([ops.muls, ops.adds])
    y2, ops2 = mttkrp_hbcsf(hs, f, 0, schedule=sched)
    c1["ops_sched"] = np.asarray([ops2.muls, ops2.adds])
    np.savez_compressed(OUT / "config1.npz", **c1)

    # -- CP-ALS fit histories --------------------------------------------
    als = {}
    grng = np.random.default_rng(5)
    fs = [grng.uniform(0.1, 1, (d, 2)) for d in (10, 12, 14)]
    dense = np.einsum("ar,br,cr->abc", *fs)
    idx = np.argwhere(dense != 0)
    t = tk.canonicalize(tk.CooTensor((10, 12, 14), idx, dense[tuple(idx.T)]))
    als["rank2/indices"], als["rank2/values"] = t.indices, t.values
    for fmt in ("coo", "csf", "bcsf", "hbcsf"):
        _, hist = tk.cp_als(t, rank=2, max_iters=12, fit_tol=1e-13, tensor_format=fmt, seed=5)
        als[f"rank2/fits_{fmt}"] = np.asarray([hh.fit for hh in hist])
        als[f"rank2/ops_{fmt}"] = np.asarray([[o.muls, o.adds] for o in hist[1].op_counts])
    rt = random_tensor(np.random.default_rng(11), (30, 25, 20), 1500)
    als["rand/indices"], als["rand/values"] = rt.indices, rt.values
    model, hist = tk.cp_als(rt, rank=8, max_iters=10, fit_tol=1e-13, seed=2)
    als["rand/fits"] = np.asarray([hh.fit for hh in hist])
    als["rand/lam"] = model.lam
    np.savez_compressed(OUT / "cp_als.npz", **als)

    meta = {"reference": "tenkit 0.1.0 (/root/reference/pkg)", "numpy": np.__version__,
            "files": sorted(p.name for p in OUT.glob("*.npz"))}
    (OUT / "MANIFEST.json").write_text(json.dumps(meta, indent=1) + "\n")
    print("wrote", meta["files"])


if __name__ == "__main__":
    main()
