"""Break down the end-to-end (host buffers) path: device-only 8-bit rate on one
and two lanes vs ils_smooth_host_u8 at several batch counts (fixed overhead
vs per-frame rate).

    python tools/e2e_probe.py
"""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2003_07504_b200 as ils  # noqa: E402
from paper_2003_07504_b200 import _lib, _runtime as rt  # noqa: E402

H, W, CH, F = 1080, 1920, 3, 64
dev = torch.device("cuda", 0)
prm = ils.SmoothParams(ils.Charbonnier(0.8, 1e-4), 1.0)
plan = rt.get_plan(CH, H, W, prm.c_params(), _lib.ILS_F32, 0)
L = _lib.lib()
wss = [torch.empty(plan.workspace_bytes, dtype=torch.uint8, device=dev) for _ in range(2)]
sts = [torch.empty(1, dtype=torch.int32, device=dev) for _ in range(2)]
f8 = torch.randint(0, 256, (F, H, W, CH), dtype=torch.uint8, device=dev)
u8 = torch.empty_like(f8)
lanes = [torch.cuda.Stream(), torch.cuda.Stream()]


def dev_u8(nlanes, frames):
    for k in range(frames):
        ln = k % nlanes
        L.ils_smooth_u8(plan.ptr, C.c_void_p(f8[k].data_ptr()), C.c_void_p(u8[k].data_ptr()), CH,
                        C.c_void_p(wss[ln].data_ptr()), C.c_void_p(lanes[ln].cuda_stream),
                        C.c_void_p(sts[ln].data_ptr()))


f32 = torch.rand((F * CH, H, W), device=dev)
u32 = torch.empty_like(f32)


def dev_f32(nlanes, frames):
    for k in range(frames):
        ln = k % nlanes
        L.ils_smooth(plan.ptr, C.c_void_p(f32[k * CH].data_ptr()), C.c_void_p(u32[k * CH].data_ptr()), H * W,
                     C.c_void_p(wss[ln].data_ptr()), C.c_void_p(lanes[ln].cuda_stream),
                     C.c_void_p(sts[ln].data_ptr()), None)


for nl in (1, 2):
    dev_f32(nl, F)
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(3):
        dev_f32(nl, F)
    torch.cuda.synchronize()
    us = (time.perf_counter() - t) * 1e6 / (3 * F)
    print(f"device f32, {nl} lane(s): {us:.1f} us/frame ({1e6 / us:.0f} fps)", flush=True)

for nl in (1, 2):
    dev_u8(nl, F)
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(3):
        dev_u8(nl, F)
    torch.cuda.synchronize()
    us = (time.perf_counter() - t) * 1e6 / (3 * F)
    print(f"device u8, {nl} lane(s): {us:.1f} us/frame ({1e6 / us:.0f} fps)", flush=True)

fh = torch.empty((F, H, W, CH), dtype=torch.uint8, pin_memory=True)
fh.copy_(f8.cpu())
uh = torch.empty_like(fh, pin_memory=True)
io = C.c_size_t()
_lib.check(L.ils_host_io_size(plan.ptr, C.byref(io)), "io")
iobuf = torch.empty(io.value, dtype=torch.uint8, device=dev)
bad = C.c_int32()
s = torch.cuda.current_stream()
for nb in (1, 4, 16, 64):
    def call():
        _lib.check(L.ils_smooth_host_u8(plan.ptr, C.c_void_p(fh.data_ptr()), C.c_void_p(uh.data_ptr()), CH, nb,
                                        C.c_void_p(wss[0].data_ptr()), C.c_void_p(iobuf.data_ptr()),
                                        C.c_void_p(s.cuda_stream), C.byref(bad)), "host_u8")
    call()
    t = time.perf_counter()
    reps = max(2, 64 // nb)
    for _ in range(reps):
        call()
    dt = (time.perf_counter() - t) / reps
    print(f"host u8 nbatches={nb}: {dt * 1e3:.3f} ms/call, {dt * 1e6 / nb:.1f} us/frame ({nb / dt:.0f} fps)", flush=True)
# host-side enqueue cost of one batch (no GPU wait): time the launches of dev_u8 alone
torch.cuda.synchronize()
torch.cuda._sleep(2_000_000_000)
t = time.perf_counter()
dev_u8(2, 16)
print(f"enqueue cost: {(time.perf_counter() - t) * 1e6 / 16:.1f} us/frame (CPU)")
torch.cuda.synchronize()
