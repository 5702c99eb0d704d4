"""Build the in-tree CUDA library libils_b200.so for sm_100a (nvcc, no JIT).

    python -m paper_2003_07504_b200.build        # or __graft_entry__.build()

The .so lands next to this file so it travels to the GPU box with the repo
snapshot (it is git-ignored, not gpurun-ignored).
"""

from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libils_b200.so")

# (source, extra defines): ils_inst.cu is compiled once per kernel family
N_ROW_SPECS = 5
N_COL_SPECS = 6
UNITS = ([("ils_api.cu", "api", [])]
         + [("ils_inst.cu", f"row_rt_{t}", [f"-DILS_INST_ROW_RT={t}"]) for t in ("float", "double")]
         + [("ils_inst.cu", f"col_rt_{t}", [f"-DILS_INST_COL_RT={t}"]) for t in ("float", "double")]
         # compile-time fp32 row plans: FFT butterflies and stencil on the packed FP32x2 pipe
         + [("ils_inst.cu", f"row_spec{i}", [f"-DILS_INST_ROW_SPEC={i}", "-DILS_PACKED_F32X2"])
            for i in range(N_ROW_SPECS)]
         + [("ils_inst.cu", f"col_spec{i}", [f"-DILS_INST_COL_SPEC={i}"]) for i in range(N_COL_SPECS)]
         + [("ils_inst.cu", "col2", ["-DILS_INST_COL2", "-DILS_PACKED_F32X2"])]
         + [("ils_inst.cu", "col3", ["-DILS_INST_COL3", "-DILS_PACKED_F32X2"])])
SOURCES = sorted({u[0] for u in UNITS})
HEADERS = ["ils_dft.cuh", "ils_fft.cuh", "ils_kernels.cuh", "ils_col2.cuh", "ils_col3.cuh", "ils_elem.cuh",
           "ils_rowroll.cuh", "ils_inst.cu"]
BASE_HEADERS = ["ils_dft.cuh", "ils_fft.cuh", "ils_kernels.cuh", "ils_rowroll.cuh"]


def _unit_deps(src, tag):
    """Files one object depends on (ils_col2.cuh only reaches the api and col2 units)."""
    deps = [src] + BASE_HEADERS
    if tag in ("api", "col2"):
        deps.append("ils_col2.cuh")
    if tag in ("api", "col3"):
        deps.append("ils_col3.cuh")
    if tag == "api":
        deps.append("ils_elem.cuh")
    deps = [os.path.join(CSRC, d) for d in deps]
    deps.append(os.path.join(ROOT, "include", "ils_b200.h"))
    deps.append(os.path.abspath(__file__))
    return deps

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17", "--expt-relaxed-constexpr",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
]
LINK_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-cudart", "static", "-ldl"]


def _nvcc():
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.sep not in cand or os.path.exists(cand)):
            return cand
    raise RuntimeError("nvcc not found")


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    deps.append(os.path.join(ROOT, "include", "ils_b200.h"))
    deps.append(os.path.abspath(__file__))
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build(force: bool = False, verbose: bool = False, extra=()) -> str:
    if not force and not _stale():
        return LIB
    objdir = os.path.join(HERE, "build_obj")
    os.makedirs(objdir, exist_ok=True)
    jobs, objs = [], []
    for src, tag, defs in UNITS:
        obj = os.path.join(objdir, tag + ".o")
        objs.append(obj)
        if not force and not extra and os.path.exists(obj):
            t = os.path.getmtime(obj)
            if all(os.path.getmtime(d) <= t for d in _unit_deps(src, tag) if os.path.exists(d)):
                continue  # object newer than everything it includes
        cmd = [_nvcc(), *NVCC_FLAGS, *extra, *defs, "-I", os.path.join(ROOT, "include"),
               "-c", os.path.join(CSRC, src), "-o", obj]
        jobs.append((tag, obj, cmd))
    nproc = max(1, min(len(jobs), os.cpu_count() or 4))
    running, failed = [], []
    for tag, obj, cmd in jobs:
        if verbose:
            print(" ".join(cmd), flush=True)
        running.append((tag, subprocess.Popen(cmd)))
        while len(running) >= nproc:
            t, p = running.pop(0)
            if p.wait() != 0:
                failed.append(t)
    for t, p in running:
        if p.wait() != 0:
            failed.append(t)
    if failed:
        raise RuntimeError(f"nvcc failed for {failed}")
    cmd = [_nvcc(), *LINK_FLAGS, *objs, "-o", LIB + ".tmp"]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    extra = [a for a in sys.argv[1:] if a.startswith("-X") or a.startswith("--")]
    print(build(force="--force" in sys.argv or bool(extra), verbose=True,
                extra=[a for a in extra if a != "--force"]))
