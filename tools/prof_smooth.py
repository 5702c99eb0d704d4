"""Run the bench's per-frame launch sequence (1080p RGB frames) for profiling.

    python tools/prof_smooth.py [--frames 4] [--group 1]
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
ap.add_argument("--frames", type=int, default=4)
ap.add_argument("--group", type=int, default=1)
ap.add_argument("--h", type=int, default=1080)
ap.add_argument("--w", type=int, default=1920)
ap.add_argument("--planes", type=int, default=3, help="planes per frame")
a = ap.parse_args()
params = ils.SmoothParams(ils.Charbonnier(0.8, 1e-4), 1.0)
F, G, H, W = a.frames, a.group, a.h, a.w
CH = a.planes
f = torch.rand((F * CH, H, W), device="cuda")
u = torch.empty_like(f)
plan = rt.get_plan(G * CH, H, W, params.c_params(), _lib.ILS_F32, 0)
ws = torch.empty(plan.workspace_bytes, dtype=torch.uint8, device="cuda")
st = torch.empty(1, dtype=torch.int32, device="cuda")
L = _lib.lib()
s = torch.cuda.current_stream().cuda_stream
for rep in range(2):
    for g0 in range(0, F, G):
        off = g0 * CH * H * W * 4
        _lib.check(L.ils_smooth(plan.ptr, C.c_void_p(f.data_ptr() + off), C.c_void_p(u.data_ptr() + off), H * W,
                                C.c_void_p(ws.data_ptr()), C.c_void_p(s), C.c_void_p(st.data_ptr()), None), "smooth")
torch.cuda.synchronize()
rt.raise_status(int(st.item()))
print("ok", plan.info)
