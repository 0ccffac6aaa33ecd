"""CPU oracle: a NumPy restatement of the reference HB-CSF / B-CSF path.

TEST INFRASTRUCTURE ONLY.  Nothing in the product package imports this
module.  Only tests/, ``__graft_entry__.smoke()`` and the ``cpu_baseline`` /
``--impl reference`` legs of bench.py use it, and only as the checker or the
timed CPU baseline — never as the thing measured or shipped.

It restates, function by function, the algorithms of the reference package
``tenkit`` 0.1.0 (/root/reference/pkg/src/tenkit, cited below as
``coo.py:L``, ``formats.py:L`` …), with plain arrays in dicts instead of the
reference's dataclasses.  Parity of this restatement is pinned against golden
vectors produced by the reference itself (tests/golden/make_golden.py, run
in the build container where /root/reference exists) and against the
reference's own known-answer cases (FIG tensor, split/schedule KATs).

Arithmetic is float64 like the reference; integer arrays use the reference's
dtypes (int64 pointers, uint32 indices).
"""
from __future__ import annotations

import math
from concurrent.futures import ThreadPoolExecutor

import numpy as np

IDX = np.uint32
PTR = np.int64
COO_LABEL, CSL_LABEL, CSF_LABEL = 0, 1, 2


# ---------------------------------------------------------------- COO layer
def lexsort_perm(indices: np.ndarray, mode_order) -> np.ndarray:
    """Stable permutation sorting rows by (col mo[0], col mo[1], ...) — coo.py:208-211.
    np.lexsort's primary key is the last one, so keys go minor..major."""
    keys = [indices[:, m] for m in reversed(tuple(mode_order))]
    return np.lexsort(keys)


def sort_entries(indices, values, mode_order):
    """sort_by_mode_order, coo.py:214-224 (without the sorted_under shortcut)."""
    p = lexsort_perm(indices, mode_order)
    return indices[p], values[p]


def canonical(indices, values):
    """canonicalize, coo.py:227-247: identity sort, np.add.reduceat over
    duplicate runs, drop exact zeros."""
    indices = np.asarray(indices, dtype=IDX)
    values = np.asarray(values, dtype=np.float64)
    if len(values) == 0:
        return indices.reshape(0, indices.shape[1] if indices.ndim == 2 else 3), values
    idx, val = sort_entries(indices, values, tuple(range(indices.shape[1])))
    first = np.ones(len(val), dtype=bool)
    first[1:] = (idx[1:] != idx[:-1]).any(axis=1)
    heads = np.nonzero(first)[0]
    sums = np.add.reduceat(val, heads)
    keep = sums != 0.0
    return idx[heads][keep], sums[keep]


def allmode_order(dims, mode):
    """coo.py:328-336: target mode, then the others by (dim, id)."""
    others = sorted((d for d in range(len(dims)) if d != mode), key=lambda d: (dims[d], d))
    return (mode, *others)


# ---------------------------------------------------------------- CSF layer
def csf_tree(indices, values, dims, mode_order):
    """build_csf, formats.py:120-168.  Returns a dict with keys
    dims, mode_order, ptrs (list), idxs (list), leaf, values, split."""
    mo = tuple(mode_order)
    n = len(mo)
    idx, val = sort_entries(np.asarray(indices, dtype=IDX), np.asarray(values, dtype=np.float64), mo)
    perm_cols = idx[:, list(mo)]
    m = len(val)
    tree = {"dims": tuple(dims), "mode_order": mo, "split": False, "values": val}
    if m == 0:
        tree["ptrs"] = [np.zeros(1, PTR) for _ in range(n - 1)]
        tree["idxs"] = [np.zeros(0, IDX) for _ in range(n - 1)]
        tree["leaf"] = np.zeros(0, IDX)
        return tree
    # node starts per level: any of the first d+1 permuted coordinates changes
    new_node = np.zeros(m, dtype=bool)
    new_node[0] = True
    starts = []
    for d in range(n - 1):
        new_node[1:] |= perm_cols[1:, d] != perm_cols[:-1, d]
        starts.append(np.nonzero(new_node)[0])
    tree["idxs"] = [perm_cols[starts[d], d].astype(IDX) for d in range(n - 1)]
    ptrs = []
    for d in range(n - 2):
        bounds = np.concatenate([starts[d], [m]])
        ptrs.append(np.searchsorted(starts[d + 1], bounds).astype(PTR))
    ptrs.append(np.concatenate([starts[n - 2], [m]]).astype(PTR))
    tree["ptrs"] = ptrs
    tree["leaf"] = perm_cols[:, n - 1].astype(IDX)
    return tree


def fiber_positions(tree):
    """formats.py:102-107."""
    pos = tree["ptrs"][0]
    for d in range(1, len(tree["mode_order"]) - 2):
        pos = tree["ptrs"][d][pos]
    return pos


def slice_nnz(tree):
    """formats.py:109-114."""
    return np.diff(tree["ptrs"][-1][fiber_positions(tree)])


def slice_labels(tree):
    """classify_slices, formats.py:194-204 (COO: 1 nnz; CSL: >=2 nnz and all
    fibers singleton; CSF otherwise)."""
    m = slice_nnz(tree)
    nf = np.diff(fiber_positions(tree))
    lab = np.full(len(tree["idxs"][0]), CSF_LABEL, dtype=np.int8)
    lab[(m >= 2) & (m == nf)] = CSL_LABEL
    lab[m == 1] = COO_LABEL
    return lab


def hbcsf(indices, values, dims, mode_order):
    """build_hbcsf, formats.py:260-299.  Returns {'coo': (indices, values),
    'csl': {slice_ptr, slice_idx, rest_idx, values}, 'csf': tree}."""
    mo = tuple(mode_order)
    idx, val = sort_entries(np.asarray(indices, dtype=IDX), np.asarray(values, dtype=np.float64), mo)
    full = csf_tree(idx, val, dims, mo)
    lab = slice_labels(full)
    per_entry = np.repeat(lab, slice_nnz(full)) if len(lab) else np.zeros(0, np.int8)
    sel = {k: per_entry == k for k in (COO_LABEL, CSL_LABEL, CSF_LABEL)}
    counts = slice_nnz(full)[lab == CSL_LABEL] if len(lab) else np.zeros(0, np.int64)
    csl = {
        "slice_ptr": np.concatenate([[0], np.cumsum(counts)]).astype(PTR),
        "slice_idx": full["idxs"][0][lab == CSL_LABEL].astype(IDX) if len(lab) else np.zeros(0, IDX),
        "rest_idx": idx[sel[CSL_LABEL]][:, list(mo[1:])].astype(IDX),
        "values": val[sel[CSL_LABEL]],
    }
    return {
        "dims": tuple(dims),
        "mode_order": mo,
        "labels": lab,
        "coo": (idx[sel[COO_LABEL]], val[sel[COO_LABEL]]),
        "csl": csl,
        "csf": csf_tree(idx[sel[CSF_LABEL]], val[sel[CSF_LABEL]], dims, mo),
    }


# ------------------------------------------------------------ balancing
def split_tree(tree, tau):
    """split_fibers on a CSF tree, balance.py:65-90.  Returns the same dict
    object when no fiber exceeds tau."""
    lp = tree["ptrs"][-1]
    sizes = np.diff(lp)
    nseg = -(-sizes // tau)
    if len(tree["values"]) == 0 or int(nseg.max(initial=1)) <= 1:
        return tree
    seg_off = np.concatenate([[0], np.cumsum(nseg)]).astype(PTR)
    total = int(seg_off[-1])
    # segment s of fiber f starts at lp[f] + (s - seg_off[f]) * tau
    owner = np.repeat(np.arange(len(sizes)), nseg)
    within = np.arange(total) - seg_off[owner]
    new_lp = np.concatenate([lp[owner] + within * tau, [lp[-1]]]).astype(PTR)
    out = dict(tree)
    out["ptrs"] = list(tree["ptrs"])
    out["idxs"] = list(tree["idxs"])
    out["idxs"][-1] = np.repeat(tree["idxs"][-1], nseg)
    out["ptrs"][-1] = new_lp
    out["ptrs"][-2] = seg_off[tree["ptrs"][-2]]
    out["split"] = True
    return out


def split_hbcsf(h, tau):
    """balance.py:93-97: only the CSF bucket is split."""
    out = dict(h)
    out["csf"] = split_tree(h["csf"], tau)
    return out


def block_schedule(tree, block_size):
    """assign_slice_blocks, balance.py:153-189, as a plain loop.  Returns
    (units int64 (U,4) = block_id, slice_pos, fiber_start, fiber_stop;
    multiplicities int64)."""
    fpos = fiber_positions(tree)
    fsz = np.diff(tree["ptrs"][-1])
    m = np.diff(tree["ptrs"][-1][fpos])
    mult = np.maximum(1, -(-m // block_size)).astype(np.int64)
    units = []
    for s in range(len(m)):
        b, e = int(fpos[s]), int(fpos[s + 1])
        if m[s] <= block_size:
            units.append((len(units), s, b, e))
            continue
        goal = math.ceil(int(m[s]) / int(mult[s]))
        run, first = 0, b
        for f in range(b, e):
            run += int(fsz[f])
            if run >= goal:
                units.append((len(units), s, first, f + 1))
                first, run = f + 1, 0
        if first < e:
            units.append((len(units), s, first, e))
    return np.array(units, dtype=np.int64).reshape(-1, 4), mult


# --------------------------------------------------------------- MTTKRP
def _check(dims, factors, mode):
    if not 0 <= mode < len(dims) or len(factors) != len(dims):
        raise ValueError("bad mode or factor count")
    ranks = {np.asarray(f).shape[1] for d, f in enumerate(factors) if d != mode}
    if len(ranks) != 1:
        raise ValueError("factor matrices disagree on rank")
    return ranks.pop()


def mttkrp_coo(indices, values, dims, factors, mode, threads=1):
    """kernels.py:109-151: sort (mode, *rest), per-entry products, segment sums.
    Returns (out, (muls, adds))."""
    r = _check(dims, factors, mode)
    n = len(dims)
    out = np.zeros((dims[mode], r))
    if len(values) == 0:
        return out, (0, 0)
    rest = [d for d in range(n) if d != mode]
    idx, val = sort_entries(np.asarray(indices, dtype=IDX), np.asarray(values, dtype=np.float64),
                            (mode, *rest))

    def span(lo, hi, buf):
        prod = val[lo:hi, None] * factors[rest[0]][idx[lo:hi, rest[0]]]
        for d in rest[1:]:
            prod = prod * factors[d][idx[lo:hi, d]]
        rows = idx[lo:hi, mode]
        heads = np.nonzero(np.concatenate([[True], rows[1:] != rows[:-1]]))[0]
        buf[rows[heads]] += np.add.reduceat(prod, heads, axis=0)

    spans = _spans(len(val), threads)
    if len(spans) == 1:
        span(*spans[0], out)
    else:
        bufs = [np.zeros_like(out) for _ in spans]
        with ThreadPoolExecutor(len(spans)) as ex:
            list(ex.map(lambda a: span(a[0][0], a[0][1], a[1]), zip(spans, bufs)))
        for b in bufs:
            out += b
    return out, ((n - 1) * len(val) * r, len(val) * r)


def _spans(n, workers):
    """kernels.py:91-95."""
    workers = max(1, min(workers, n))
    cuts = [round(w * n / workers) for w in range(workers + 1)]
    return [(a, b) for a, b in zip(cuts[:-1], cuts[1:]) if b > a]


def mttkrp_csl(csl, dims, mode_order, factors, mode, threads=1):
    """kernels.py:189-226."""
    r = _check(dims, factors, mode)
    n = len(dims)
    out = np.zeros((dims[mode], r))
    vals = csl["values"]
    if len(vals) == 0:
        return out, (0, 0)
    sp, si, rest = csl["slice_ptr"], csl["slice_idx"], csl["rest_idx"]

    def span(a, b, buf):
        lo, hi = int(sp[a]), int(sp[b])
        prod = vals[lo:hi, None] * factors[mode_order[1]][rest[lo:hi, 0]]
        for c in range(1, n - 1):
            prod = prod * factors[mode_order[c + 1]][rest[lo:hi, c]]
        buf[si[a:b]] += np.add.reduceat(prod, sp[a:b] - lo, axis=0)

    spans = _spans(len(si), threads)
    if len(spans) == 1:
        span(*spans[0], out)
    else:
        bufs = [np.zeros_like(out) for _ in spans]
        with ThreadPoolExecutor(len(spans)) as ex:
            list(ex.map(lambda a: span(a[0][0], a[0][1], a[1]), zip(spans, bufs)))
        for b in bufs:
            out += b
    return out, ((n - 1) * len(vals) * r, len(vals) * r)


def mttkrp_csf(tree, factors, mode):
    """kernels.py:154-186: bottom-up partial sums, one R-vector per node."""
    mo = tree["mode_order"]
    if mo[0] != mode:
        raise ValueError("tree built for another mode")
    dims = tree["dims"]
    r = _check(dims, factors, mode)
    n = len(dims)
    out = np.zeros((dims[mode], r))
    m = len(tree["values"])
    if m == 0:
        return out, (0, 0)
    pf = [factors[k] for k in mo]
    part = tree["values"][:, None] * pf[n - 1][tree["leaf"]]
    muls = adds = m * r
    part = np.add.reduceat(part, tree["ptrs"][n - 2][:-1], axis=0)
    for d in range(n - 2, 0, -1):
        part = part * pf[d][tree["idxs"][d]]
        muls += len(tree["idxs"][d]) * r
        if d < n - 2:
            adds += len(tree["idxs"][d]) * r
        part = np.add.reduceat(part, tree["ptrs"][d - 1][:-1], axis=0)
    out[tree["idxs"][0]] = part
    adds += len(tree["idxs"][0]) * r
    return out, (muls, adds)


def _unit(tree, pf, f0, f1):
    """_unit_partial, kernels.py:256-286."""
    n = len(tree["mode_order"])
    lp = tree["ptrs"][n - 2]
    lo, hi = int(lp[f0]), int(lp[f1])
    part = tree["values"][lo:hi, None] * pf[n - 1][tree["leaf"][lo:hi]]
    mul_nodes = add_nodes = hi - lo
    part = np.add.reduceat(part, lp[f0:f1] - lo, axis=0) * pf[n - 2][tree["idxs"][n - 2][f0:f1]]
    mul_nodes += f1 - f0
    a_lo, a_hi = f0, f1
    for d in range(n - 3, 0, -1):
        p = tree["ptrs"][d]
        a = int(np.searchsorted(p, a_lo, side="right")) - 1
        b = int(np.searchsorted(p, a_hi, side="left"))
        part = np.add.reduceat(part, np.clip(p[a:b], a_lo, a_hi) - a_lo, axis=0)
        part = part * pf[d][tree["idxs"][d][a:b]]
        mul_nodes += b - a
        add_nodes += b - a
        a_lo, a_hi = a, b
    return part.sum(axis=0), mul_nodes, add_nodes


def mttkrp_scheduled(tree, units, factors, mode, threads=1):
    """kernels.py:289-342 (units: int64 (U,4) array)."""
    mo = tree["mode_order"]
    dims = tree["dims"]
    r = _check(dims, factors, mode)
    out = np.zeros((dims[mode], r))
    if len(tree["values"]) == 0:
        return out, (0, 0)
    pf = [factors[k] for k in mo]
    rows = tree["idxs"][0]

    def run(us, buf):
        mn = an = 0
        for u in us:
            vec, a, b = _unit(tree, pf, int(u[2]), int(u[3]))
            buf[rows[int(u[1])]] += vec
            mn += a
            an += b + 1
        return mn, an

    if threads <= 1:
        mn, an = run(units, out)
    else:
        bufs = [np.zeros_like(out) for _ in range(threads)]
        chunks = [units[w::threads] for w in range(threads)]
        with ThreadPoolExecutor(threads) as ex:
            res = list(ex.map(run, chunks, bufs))
        for b in bufs:
            out += b
        mn = sum(x for x, _ in res)
        an = sum(y for _, y in res)
    return out, (mn * r, an * r)


def mttkrp_hbcsf(h, factors, mode, units=None, threads=1):
    """kernels.py:229-253: sum of the three bucket kernels."""
    dims, mo = h["dims"], h["mode_order"]
    y1, k1 = mttkrp_coo(*h["coo"], dims, factors, mode, threads)
    y2, k2 = mttkrp_csl(h["csl"], dims, mo, factors, mode, threads)
    if units is None:
        y3, k3 = mttkrp_csf(h["csf"], factors, mode)
    else:
        y3, k3 = mttkrp_scheduled(h["csf"], units, factors, mode, threads)
    return y1 + y2 + y3, (k1[0] + k2[0] + k3[0], k1[1] + k2[1] + k3[1])


def row_deviation(y, ref):
    """max_i ||y_i - o_i|| / (1 + ||o_i||)  (cli.py:231-234)."""
    num = np.linalg.norm(np.asarray(y, dtype=np.float64) - ref, axis=-1)
    return float((num / (1.0 + np.linalg.norm(ref, axis=-1))).max(initial=0.0))


# --------------------------------------------------------------- CP-ALS
def _gram(f):
    g = f.T @ f
    return (g + g.T) * 0.5


def _pinv(g):
    w, v = np.linalg.eigh((g + g.T) * 0.5)
    tol = g.shape[0] * np.finfo(np.float64).eps * max(float(w[-1]), 0.0)
    inv = np.where(w > tol, 1.0 / np.where(w > tol, w, 1.0), 0.0)
    out = (v * inv) @ v.T
    return (out + out.T) * 0.5


def cp_als(indices, values, dims, rank=32, max_iters=50, fit_tol=1e-8, seed=0):
    """cp_als with the hbcsf format, cpd.py:198-271 (fits only).  Returns the
    list of fits (iteration 0 first) and the final normalised factors/lambda."""
    idx, val = canonical(indices, values)
    reps = [hbcsf(idx, val, dims, allmode_order(dims, m)) for m in range(len(dims))]
    rng = np.random.default_rng(seed)
    fac = [rng.random((d, rank)) for d in dims]
    grams = [_gram(f) for f in fac]
    nx = float(np.linalg.norm(val))
    last = len(dims) - 1

    def fit_of(y):
        had = np.ones((rank, rank))
        for g in grams:
            had = had * g
        inner = float((y * fac[last]).sum())
        return 1.0 - math.sqrt(max(nx * nx + float(had.sum()) - 2.0 * inner, 0.0)) / nx

    fits = [fit_of(mttkrp_hbcsf(reps[last], fac, last)[0])]
    lam = None
    for _ in range(max_iters):
        y = None
        for mode in range(len(dims)):
            y, _ = mttkrp_hbcsf(reps[mode], fac, mode)
            v = np.ones((rank, rank))
            for d, g in enumerate(grams):
                if d != mode:
                    v = v * g
            fac[mode] = y @ _pinv(v)
            grams[mode] = _gram(fac[mode])
        new = fit_of(y)
        lam = np.ones(rank)
        for d in range(len(dims)):
            nrm = np.linalg.norm(fac[d], axis=0)
            nrm = np.where(nrm > 0.0, nrm, 1.0)
            fac[d] = fac[d] / nrm
            grams[d] = grams[d] / np.outer(nrm, nrm)
            lam = lam * nrm
        delta = new - fits[-1]
        fits.append(new)
        if abs(delta) < fit_tol:
            break
    return fits, fac, lam
