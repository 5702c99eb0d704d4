"""Build a variant of libils_b200.so with extra nvcc flags into variants/<name>.so
(git-ignored, travels to the GPU box); select it at run time with ILS_LIB.

    python tools/build_variant.py kb4 -DILS_STENCIL_ROWS=4
"""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2003_07504_b200 import build as B  # noqa: E402

name, flags = sys.argv[1], sys.argv[2:]
out_dir = os.path.join(B.ROOT, "variants")
obj_dir = os.path.join("/tmp", "ils_variant_" + name)
os.makedirs(out_dir, exist_ok=True)
os.makedirs(obj_dir, exist_ok=True)
procs, objs = [], []
for src, tag, defs in B.UNITS:
    obj = os.path.join(obj_dir, tag + ".o")
    objs.append(obj)
    cmd = [B._nvcc(), *B.NVCC_FLAGS, *flags, *defs, "-I", os.path.join(B.ROOT, "include"), "-c",
           os.path.join(B.CSRC, src), "-o", obj]
    procs.append(subprocess.Popen(cmd))
    while sum(p.poll() is None for p in procs) >= (os.cpu_count() or 4):
        procs[[p.poll() is None for p in procs].index(True)].wait()
if any(p.wait() != 0 for p in procs):
    sys.exit("nvcc failed")
lib = os.path.join(out_dir, name + ".so")
subprocess.run([B._nvcc(), *B.LINK_FLAGS, *objs, "-o", lib], check=True)
print(lib)
