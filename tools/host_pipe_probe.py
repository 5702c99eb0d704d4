"""Python replica of ils_smooth_host_u8's pipeline (tools only): pinned 8-bit
RGB frames in, H2D on one stream, compute on L lanes, D2H on one stream,
NS device I/O slots.  Timeline per batch from CUDA events, and variants."""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2003_07504_b200 as ils  # noqa: E402
from paper_2003_07504_b200 import _lib, _runtime as rt  # noqa: E402

H, W, CH, F = 1080, 1920, 3, 64
prm = ils.SmoothParams(ils.Charbonnier(0.8, 1e-4), 1.0)
plan = rt.get_plan(CH, H, W, prm.c_params(), _lib.ILS_F32, 0)
L = _lib.lib()
fh = torch.randint(0, 256, (F, H, W, CH), dtype=torch.uint8).pin_memory()
uh = torch.empty_like(fh).pin_memory()
NSMAX = 8
fs = torch.empty((NSMAX, H, W, CH), dtype=torch.uint8, device="cuda")
us = torch.empty_like(fs)
wss = [torch.empty(plan.workspace_bytes, dtype=torch.uint8, device="cuda") for _ in range(4)]
st = torch.empty(16, dtype=torch.int32, device="cuda")
h2ds = [torch.cuda.Stream() for _ in range(4)]
d2hs = [torch.cuda.Stream() for _ in range(4)]
lanes = [torch.cuda.Stream() for _ in range(4)]


def run(nl, ns, copies=True, timeline=False, nh=1, split=1):
    ev_in = [torch.cuda.Event() for _ in range(ns)]
    ev_comp = [torch.cuda.Event() for _ in range(ns)]
    ev_out = [torch.cuda.Event() for _ in range(ns)]
    tl = []
    for k in range(F):
        sl, ln = k % ns, k % nl
        h2d, d2h = h2ds[k % nh], d2hs[k % nh]
        t = [torch.cuda.Event(enable_timing=True) for _ in range(6)] if timeline else None
        if k >= ns:
            h2d.wait_event(ev_comp[sl])
        if t: t[0].record(h2d)
        if copies:
            if split == 1:
                with torch.cuda.stream(h2d):
                    fs[sl].copy_(fh[k], non_blocking=True)
            else:  # the frame's rows in `split` parts on as many streams
                hh = H // split
                for q in range(split):
                    sq = h2ds[q]
                    if q:
                        sq.wait_stream(h2d)
                    with torch.cuda.stream(sq):
                        fs[sl, q * hh:(q + 1) * hh].copy_(fh[k, q * hh:(q + 1) * hh], non_blocking=True)
                    if q:
                        h2d.wait_stream(sq)
        if t: t[1].record(h2d)
        ev_in[sl].record(h2d)
        lanes[ln].wait_event(ev_in[sl])
        if k >= ns:
            lanes[ln].wait_event(ev_out[sl])
        if t: t[2].record(lanes[ln])
        L.ils_smooth_u8(plan.ptr, C.c_void_p(fs[sl].data_ptr()), C.c_void_p(us[sl].data_ptr()), CH,
                        C.c_void_p(wss[ln].data_ptr()), C.c_void_p(lanes[ln].cuda_stream), C.c_void_p(st[sl:].data_ptr()))
        if t: t[3].record(lanes[ln])
        ev_comp[sl].record(lanes[ln])
        d2h.wait_event(ev_comp[sl])
        if t: t[4].record(d2h)
        if copies:
            with torch.cuda.stream(d2h):
                uh[k].copy_(us[sl], non_blocking=True)
        if t: t[5].record(d2h)
        ev_out[sl].record(d2h)
        if t: tl.append(t)
    torch.cuda.synchronize()
    return tl


for nl, ns, nh, split in [(2, 4, 1, 1), (2, 4, 2, 1), (2, 8, 2, 1), (2, 8, 4, 1), (2, 4, 1, 2), (2, 4, 1, 4)]:
    run(nl, ns, True, nh=nh, split=split)
    t0 = time.perf_counter()
    for _ in range(3):
        run(nl, ns, True, nh=nh, split=split)
    us_f = (time.perf_counter() - t0) * 1e6 / (3 * F)
    print(f"lanes {nl} slots {ns} copy streams {nh} split {split}: {us_f:.1f} us/frame ({1e6 / us_f:.0f} fps)",
          flush=True)

