"""Build libhbk.so in-tree for sm_100a (``python -m paper_1904_03329_b200.build``)."""
from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
SOURCES = ["csrc/build.cu", "csrc/mttkrp.cu", "csrc/als.cu", "csrc/frostt.cpp", "csrc/stage.cpp"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-O3",
         "--expt-relaxed-constexpr", "-Wno-deprecated-gpu-targets", f"-I{ROOT / 'include'}"]


def nvcc() -> str:
    cand = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not Path(cand).exists():
        raise RuntimeError("nvcc not found")
    return cand


def build(verbose: bool = False, jobs: int | None = None) -> Path:
    out = PKG / "libhbk.so"
    objs = []
    env = dict(os.environ)
    procs = []
    for src in SOURCES:
        obj = PKG / "csrc" / (Path(src).stem + ".o")
        cmd = [nvcc(), *ARCH, *FLAGS, "-c", str(PKG / src), "-o", str(obj)]
        if verbose:
            print(" ".join(cmd), flush=True)
        procs.append((subprocess.Popen(cmd, env=env, stdout=subprocess.PIPE, stderr=subprocess.STDOUT), src))
        objs.append(obj)
    for p, src in procs:
        log, _ = p.communicate()
        if p.returncode != 0:
            raise RuntimeError(f"nvcc failed on {src}:\n{log.decode(errors='replace')}")
    cmd = [nvcc(), *ARCH, "-shared", "-o", str(out), *map(str, objs), "-lcudart_static", "-lrt",
           "-lpthread", "-ldl"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"link failed:\n{res.stdout}\n{res.stderr}")
    for o in objs:
        o.unlink(missing_ok=True)
    return out


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
