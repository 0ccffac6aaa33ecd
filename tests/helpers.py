"""Shared fixtures for the parity tests (golden-case iteration, factors)."""
from __future__ import annotations

import hashlib
import re
import zlib

import numpy as np

from conftest import golden

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


def fig_arrays():
    rows = [line.split() for line in FIG_TEXT.strip().splitlines()]
    idx = np.array([[int(x) - 1 for x in r[:3]] for r in rows], dtype=np.uint32)
    vals = np.array([float(r[3]) for r in rows])
    return idx, vals


def digest(a: np.ndarray) -> str:
    a = np.ascontiguousarray(a)
    return hashlib.sha256(a.dtype.str.encode() + str(a.shape).encode() + a.tobytes()).hexdigest()


def golden_factors(key: str, dims, rank):
    """Same factors tests/golden/make_golden.py fed the reference."""
    rng = np.random.default_rng(zlib.crc32(key.encode()))
    return [rng.random((d, rank)).astype(np.float32).astype(np.float64) for d in dims]


def cases():
    """Golden tensors of formats_kernels.npz: (key, indices, values, dims)."""
    g = golden("formats_kernels")
    keys = sorted({k.split("/")[0] for k in g})
    for key in keys:
        yield key, g[f"{key}/indices"], g[f"{key}/values"], tuple(int(d) for d in g[f"{key}/dims"])


def mode_blocks(key: str):
    """(mode, prefix) of a golden case."""
    g = golden("formats_kernels")
    modes = sorted({int(m.group(1)) for k in g for m in [re.match(rf"{key}/m(\d+)/", k)] if m})
    return [(m, f"{key}/m{m}") for m in modes]


def cfg_blocks(prefix: str):
    g = golden("formats_kernels")
    cfgs = sorted({int(m.group(1)) for k in g for m in [re.match(rf"{re.escape(prefix)}/cfg(\d+)/", k)] if m})
    return [(c, f"{prefix}/cfg{c}", tuple(int(x) for x in g[f"{prefix}/cfg{c}/cfg"])) for c in cfgs]


def rank_blocks(prefix: str):
    g = golden("formats_kernels")
    rs = sorted({int(m.group(1)) for k in g for m in [re.match(rf"{re.escape(prefix)}/r(\d+)/", k)] if m})
    return [(r, f"{prefix}/r{r}") for r in rs]


def row_dev(y, ref) -> float:
    """Reference row metric max ||y_i - o_i|| / (1 + ||o_i||) (cli.py:231-234)."""
    num = np.linalg.norm(np.asarray(y, dtype=np.float64) - ref, axis=-1)
    return float((num / (1.0 + np.linalg.norm(ref, axis=-1))).max(initial=0.0))
