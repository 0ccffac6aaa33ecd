"""bench.py keeps the driver's contract: one JSON line with the required keys
(both arms), sane values, and the roofline / cpu_baseline / e2e / clocks /
gpu_launches objects this tier adds.  Small scale so it runs in seconds."""
from __future__ import annotations

import json
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
             "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config"}


def _run(*args):
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), *args], capture_output=True,
                         text=True, cwd=ROOT, timeout=900)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout[-3000:]
    return json.loads(lines[0])


def test_gpu_arm_json_line():
    d = _run("--steps", "3", "--warmup", "3", "--scale", "0.05", "--cpu-sample-nnz", "20000")
    assert BASE_KEYS <= d.keys()
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] == 3
    assert d["value"] > 0 and d["ms_per_step"] > 0 and d["higher_is_better"] is True
    assert d["config"]["workload"].startswith("nell-2")
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and 0 < r["frac"] < 1
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["value"] > 0
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] == 3 * sum(r["launches_per_mode"])
    assert "sm_mhz" in d["clocks"] and "reasons" in d["clocks"]
    p = d["parity"]
    assert p["format_bit_exact"] is True and p["max_row_dev"] <= 1e-4
    assert d["e2e"]["pinned_fp32"]["value"] > 0
    assert d["cpd"]["ms_per_sweep"] > 0 and len(d["cpd"]["fits"]) >= 2


def test_two_ranks_on_one_gpu():
    """--gpus 2 without torchrun: bench.py launches the ranks itself (gloo,
    sharing the one GPU here) and reports the 2-rank job."""
    d = _run("--gpus", "2", "--steps", "3", "--warmup", "3", "--scale", "0.05", "--cpd", "none")
    assert d["n_gpus"] == 2 and len(d["config"]["ranks"]) == 2
    assert d["config"]["workload"].startswith("flickr-3d")
    assert d["config"]["parallelism"] == "slice-sharded dp2"
    assert d["with_output_allgather"]["value"] > 0
    assert d["value"] > 0


def test_reference_arm_json_line():
    d = _run("--impl", "reference", "--steps", "2", "--warmup", "1", "--scale", "0.05",
             "--cpu-sample-nnz", "20000")
    assert BASE_KEYS <= d.keys() and d["impl"] == "reference"
    assert d["value"] > 0 and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["value"] == d["value"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["cpu_baseline"]["threads1_value"] > 0
    assert d["native_libraries"].startswith("none")
