"""Device-resident timing of the 8-bit path vs the fp32-plane path (1080p RGB, N=4).

    python tools/time_u8.py [--frames 16]
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
ap.add_argument("--frames", type=int, default=16)
a = ap.parse_args()
H, W, CH, F = 1080, 1920, 3, a.frames
dev = torch.device("cuda", 0)
prm = ils.SmoothParams(ils.Charbonnier(0.8, 1e-4), 1.0)
plan = rt.get_plan(CH, H, W, prm.c_params(), _lib.ILS_F32, 0)
L = _lib.lib()
ws = torch.empty(plan.workspace_bytes, dtype=torch.uint8, device=dev)
st = torch.empty(1, dtype=torch.int32, device=dev)
f8 = torch.randint(0, 256, (F, H, W, CH), dtype=torch.uint8, device=dev)
u8 = torch.empty_like(f8)
f32 = torch.rand((F * CH, H, W), device=dev)
u32 = torch.empty_like(f32)
s = torch.cuda.current_stream().cuda_stream


def run_u8(k):
    L.ils_smooth_u8(plan.ptr, C.c_void_p(f8[k].data_ptr()), C.c_void_p(u8[k].data_ptr()), CH, C.c_void_p(ws.data_ptr()),
                    C.c_void_p(s), C.c_void_p(st.data_ptr()))


def run_f32(k):
    L.ils_smooth(plan.ptr, C.c_void_p(f32[k * CH].data_ptr()), C.c_void_p(u32[k * CH].data_ptr()), H * W,
                 C.c_void_p(ws.data_ptr()), C.c_void_p(s), C.c_void_p(st.data_ptr()), None)


def run_pass(mode, p):
    # one pass of the sequence on frame 0
    L.ils_launch_pass(plan.ptr, p, C.c_void_p(f32.data_ptr()), C.c_void_p(u32.data_ptr()), H * W,
                      C.c_void_p(ws.data_ptr()), C.c_void_p(s), C.c_void_p(st.data_ptr()))


for name, fn in (("f32", run_f32), ("u8", run_u8)):
    for _ in range(2):
        for k in range(F):
            fn(k)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda._sleep(100_000_000)
    e0.record()
    for _ in range(5):
        for k in range(F):
            fn(k)
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / (5 * F)
    print(f"{name}: {us:.1f} us/frame  ({1e6 / us:.0f} fps, one lane)")
