"""CP-ALS fit history of the fused fp32 path (R=32: fast MTTKRP + tensor-core
row update) against the fp64 MTTKRP path on nell-2 (first four sweeps).
    python scripts/fit_compare.py"""
import sys, numpy as np
sys.path.insert(0, '.')
import paper_1904_03329_b200 as hb
from paper_1904_03329_b200.generate import config_tensor
t = config_tensor("nell-2")
m32, h32 = hb.cp_als(t, rank=32, max_iters=4, fit_tol=0.0, seed=5)
m64, h64 = hb.cp_als(t, rank=32, max_iters=4, fit_tol=0.0, seed=5, mttkrp_precision="fp64")
print("fp32", [h.fit for h in h32]); print("fp64", [h.fit for h in h64])
