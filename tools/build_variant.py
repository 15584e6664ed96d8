"""Build an experimental variant of the library with extra nvcc defines into
paper_2104_00792_b200/exp/<name>.so (git-ignored; travels with gpurun).  Load it
with HG_LIB=<path> (paper_2104_00792_b200/_lib.py honours the override).
usage: python tools/build_variant.py NAME -DFOO=1 ..."""
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2104_00792_b200 import _build as B  # noqa: E402

name, defs = sys.argv[1], sys.argv[2:]
out_dir = os.path.join(B.HERE, "exp", name)
os.makedirs(out_dir, exist_ok=True)
nvcc = B._nvcc()


def one(src):
    obj = os.path.join(out_dir, os.path.basename(src).replace(".cu", ".o"))
    r = subprocess.run([nvcc, *B.ARCH, *B.FLAGS, *defs, "-c", src, "-o", obj], capture_output=True, text=True)
    if r.returncode:
        raise SystemExit(r.stderr)
    return obj


with ThreadPoolExecutor(8) as pool:
    objs = list(pool.map(one, B._sources()))
lib = os.path.join(B.HERE, "exp", f"{name}.so")
r = subprocess.run([nvcc, *B.ARCH, "-shared", "-o", lib, *objs, "-cudart=static"], capture_output=True, text=True)
if r.returncode:
    raise SystemExit(r.stderr)
print(lib)
