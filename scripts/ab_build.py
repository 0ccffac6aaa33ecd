"""Build a variant of libhbk.so with extra -D flags for same-box A/B timing
(load it with HBK_LIB=<path>):
    python scripts/ab_build.py ab/libhbk_pf0.so -DHBK_CSL_PREFETCH=0"""
import subprocess
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1904_03329_b200 import build as B

out = Path(sys.argv[1]).resolve()
defs = sys.argv[2:]
out.parent.mkdir(parents=True, exist_ok=True)
objs, procs = [], []
for src in B.SOURCES:
    obj = out.parent / (out.stem + "_" + Path(src).stem + ".o")
    procs.append(subprocess.Popen([B.nvcc(), *B.ARCH, *B.FLAGS, *defs, "-c", str(B.PKG / src), "-o", str(obj)]))
    objs.append(obj)
assert all(p.wait() == 0 for p in procs)
subprocess.check_call([B.nvcc(), *B.ARCH, "-shared", "-o", str(out), *map(str, objs), "-lcudart_static",
                       "-lrt", "-lpthread", "-ldl"])
for o in objs:
    o.unlink()
print(out)
