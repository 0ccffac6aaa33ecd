"""Pure-Python loop oracles for small cases — TEST INFRASTRUCTURE ONLY.

Independent of both the reference's vectorised code and tenkit_port: dict
accumulation and per-entry loops, in the spirit of the reference's own
tests/helpers.py (reference_mttkrp :55-65, entry_map :68-73,
group_sizes :76-82).
"""
from __future__ import annotations

import numpy as np


def mttkrp_entries(indices, values, dims, factors, mode):
    """out[i_mode] += v * prod_{d != mode} F_d[i_d], one entry at a time."""
    rank = None
    for d, f in enumerate(factors):
        if d != mode:
            rank = np.asarray(f).shape[1]
            break
    out = np.zeros((dims[mode], rank))
    for row, v in zip(np.asarray(indices), np.asarray(values)):
        acc = np.full(rank, float(v))
        for d, i in enumerate(row):
            if d != mode:
                acc = acc * factors[d][int(i)]
        out[int(row[mode])] += acc
    return out


def entry_map(indices, values):
    """Coordinate -> summed value, exact zeros dropped."""
    acc = {}
    for row, v in zip(np.asarray(indices), np.asarray(values)):
        key = tuple(int(i) for i in row)
        acc[key] = acc.get(key, 0.0) + float(v)
    return {k: v for k, v in acc.items() if v != 0.0}


def group_sizes(indices, mode_order, depth):
    """Nonzeros per distinct prefix of length ``depth`` under mode_order."""
    counts = {}
    for row in np.asarray(indices):
        key = tuple(int(row[m]) for m in mode_order[:depth])
        counts[key] = counts.get(key, 0) + 1
    return list(counts.values())
