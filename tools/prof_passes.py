"""Launch each pass of the 1080p RGB plan a few times (for ncu / launch lists).

    python tools/prof_passes.py [--reps 3] [--h 1080 --w 1920 --planes 3]
"""
import argparse
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2003_07504_b200 as ils  # noqa: E402
from paper_2003_07504_b200 import _lib, _runtime as rt  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--h", type=int, default=1080)
ap.add_argument("--w", type=int, default=1920)
ap.add_argument("--planes", type=int, default=3)
ap.add_argument("--full", action="store_true", help="also run one full ils_smooth")
a = ap.parse_args()
params = ils.SmoothParams(ils.Charbonnier(0.8, 1e-4), 1.0)
f = torch.rand((a.planes, a.h, a.w), device="cuda")
u = torch.empty_like(f)
plan = rt.get_plan(a.planes, a.h, a.w, params.c_params(), _lib.ILS_F32, 0)
ws = torch.empty(plan.workspace_bytes, dtype=torch.uint8, device="cuda")
st = torch.empty(1, dtype=torch.int32, device="cuda")
L = _lib.lib()
s = torch.cuda.current_stream().cuda_stream
for p in (0, 1, 2, 3):
    for _ in range(a.reps):
        _lib.check(L.ils_launch_pass(plan.ptr, p, C.c_void_p(f.data_ptr()), C.c_void_p(u.data_ptr()), a.h * a.w,
                                     C.c_void_p(ws.data_ptr()), C.c_void_p(s), C.c_void_p(st.data_ptr())), "pass")
if a.full:
    ils.smooth_batch(f, params)
torch.cuda.synchronize()
print("ok", plan.info)
