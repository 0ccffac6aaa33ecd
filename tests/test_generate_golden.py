"""The restated reference generator (oracle/ref_generate.py,
generate.py:62-115) against tensors the reference itself produced
(tests/golden/generate.npz, config1.npz).  Canonicalisation uses the pinned
oracle."""
from __future__ import annotations

import numpy as np
import pytest

from conftest import golden
from oracle import tenkit_port as P
from oracle.ref_generate import generate_raw as _generate_raw

CASES = ["skew12", "skew0_4d", "dense_slices", "overflow"]


@pytest.mark.parametrize("key", CASES)
def test_generator_matches_reference(key):
    g = golden("generate")
    a = [int(x) for x in g[f"{key}/args"]]
    dims, nnz, seed = tuple(a[:-2]), a[-2], a[-1]
    _, idx, vals = _generate_raw(dims, nnz, float(g[f"{key}/skew"]), seed)
    ci, cv = P.canonical(idx.astype(np.uint32), vals)
    assert np.array_equal(ci, g[f"{key}/indices"])
    assert np.array_equal(cv.view(np.int64), g[f"{key}/values"].view(np.int64))


def test_config1_generator_bit_exact():
    g = golden("config1")
    _, idx, vals = _generate_raw((1000, 1000, 1000), 100_000, 0.0, 0)
    ci, cv = P.canonical(idx.astype(np.uint32), vals)
    assert np.array_equal(ci, g["indices"])
    assert np.array_equal(cv, g["values"])


def test_generator_argument_errors():
    with pytest.raises(ValueError):
        _generate_raw((3, 3), 1, 1.0, 0)
    with pytest.raises(ValueError):
        _generate_raw((3, 3, 3), 1, -1.0, 0)
    with pytest.raises(ValueError):
        _generate_raw((3, 3, 3), 28, 1.0, 0)
