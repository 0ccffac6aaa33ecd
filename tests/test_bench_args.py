"""bench.py's workload defaults (CPU): nell-2 (configs[1]) is the N=1
headline; at N>1 the metric's multi-GPU configuration flickr-3d leads and
nell-2 rides along in ``also`` so every N of a scaling run has the N=1
config too."""
from __future__ import annotations

import importlib.util
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def _args(monkeypatch, *argv, world=None):
    spec = importlib.util.spec_from_file_location("bench_under_test", ROOT / "bench.py")
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    monkeypatch.setattr(sys, "argv", ["bench.py", *argv])
    if world is None:
        monkeypatch.delenv("WORLD_SIZE", raising=False)
    else:
        monkeypatch.setenv("WORLD_SIZE", str(world))
    return mod.parse_args()


def test_single_gpu_defaults(monkeypatch):
    a = _args(monkeypatch)
    assert a.config == "nell-2" and a.also == ["flickr-3d", "delicious-3d"] and a.cpd == "nell-1"


def test_multi_gpu_defaults_carry_the_headline(monkeypatch):
    for argv, world in ((("--gpus", "8"), None), ((), 4)):
        a = _args(monkeypatch, *argv, world=world)
        assert a.config == "flickr-3d" and a.also == ["nell-2"]


def test_scaled_runs_add_nothing(monkeypatch):
    a = _args(monkeypatch, "--gpus", "2", "--scale", "0.05")
    assert a.config == "flickr-3d" and a.also == []
