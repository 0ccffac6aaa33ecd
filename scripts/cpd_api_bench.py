"""cp_als (R=32) sweep times on the config tensors (1 GPU)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1904_03329_b200 as hb
from paper_1904_03329_b200.generate import config_tensor

for c in (sys.argv[1:] or ["nell-2", "nell-1"]):
    t = config_tensor(c)
    m, h = hb.cp_als(t, rank=32, max_iters=5, fit_tol=0.0, seed=1)
    print(c, "sweep ms", [round(sum(x.mode_seconds) * 1e3, 2) for x in h[1:]], "fit", h[-1].fit,
          flush=True)
