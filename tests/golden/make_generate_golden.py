"""Golden outputs of the reference's generate_tensor (generate.py:62-115).

Run in the build container (imports tenkit from /root/reference):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_generate_golden.py
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")
import tenkit as tk  # noqa: E402

CASES = {
    "skew12": ((50, 40, 30), 3000, 1.2, 7),
    "skew0_4d": ((9, 8, 7, 6), 1500, 0.0, 3),
    "dense_slices": ((4, 3, 3), 30, 2.0, 1),   # near-complete slices (permutation branch)
    "overflow": ((6, 2, 2), 20, 3.0, 5),       # multinomial overflow pushed to later slices
}


def main():
    out = {}
    for key, (dims, nnz, skew, seed) in CASES.items():
        t = tk.generate_tensor(dims, nnz, skew=skew, seed=seed)
        out[f"{key}/indices"] = t.indices
        out[f"{key}/values"] = t.values
        out[f"{key}/args"] = np.asarray([*dims, nnz, seed], dtype=np.int64)
        out[f"{key}/skew"] = np.asarray(skew)
    np.savez_compressed(Path(__file__).resolve().parent / "generate.npz", **out)
    print("wrote", sorted(CASES))


if __name__ == "__main__":
    main()
