"""Build a variant of libils_b200.so with extra nvcc flags into variants/<name>.so
(git-ignored, travels to the GPU box); select it at run time with ILS_LIB.

    python tools/build_variant.py kb4 -DILS_STENCIL_ROWS=4
    python tools/build_variant.py pk --only row_spec1,col2 -DILS_PACKED_F32X2

--only recompiles just the listed units with the flags and links the rest
from the default build's objects (paper_2003_07504_b200/build_obj).
"""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2003_07504_b200 import build as B  # noqa: E402

args = sys.argv[1:]
name = args.pop(0)
only = None
if "--only" in args:
    i = args.index("--only")
    only = set(args[i + 1].split(","))
    del args[i:i + 2]
flags = args
out_dir = os.path.join(B.ROOT, "variants")
obj_dir = os.path.join("/tmp", "ils_variant_" + name)
os.makedirs(out_dir, exist_ok=True)
os.makedirs(obj_dir, exist_ok=True)
if only:
    B.build()  # the default objects the variant links against
procs, objs = [], []
for src, tag, defs in B.UNITS:
    if only and tag not in only:
        objs.append(os.path.join(B.HERE, "build_obj", tag + ".o"))
        continue
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
