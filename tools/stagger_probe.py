"""Lane stagger probe: the bench's two lanes start in phase (both run their
first row pass, then both their column pass, ...).  Offset lane 1 by k passes
of lane 0's first frame (per-pass launches + an event) so row passes of one
lane meet column passes of the other; 32 1080p RGB frames per step."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2003_07504_b200 as ils  # noqa: E402
from paper_2003_07504_b200 import _lib, _runtime as rt  # noqa: E402

H, W, F, CH, ITERS = 1080, 1920, 32, 3, 4
params = ils.SmoothParams(ils.Charbonnier(0.8, 1e-4), 1.0, iters=ITERS)
f = torch.rand((F * CH, H, W), device="cuda")
u = torch.empty_like(f)
L = _lib.lib()
plan = rt.get_plan(CH, H, W, params.c_params(), _lib.ILS_F32, 0)
wss = [torch.empty(plan.workspace_bytes, dtype=torch.uint8, device="cuda") for _ in range(2)]
st = torch.empty(2, dtype=torch.int32, device="cuda")
order = [0, 1]
for n in range(1, ITERS):
    cur = 0 if n % 2 else 4
    order += [2 | cur, 1 | (cur ^ 4)]
order += [3 | (0 if ITERS % 2 else 4)]
ps = H * W
for k in range(0, 6):
    main, l1 = torch.cuda.Stream(), torch.cuda.Stream()
    lanes = [main, l1]

    def step():
        l1.wait_stream(main)
        ev = torch.cuda.Event()
        for fr in range(F):
            ln = fr % 2
            off = fr * CH * ps * 4
            if fr == 0 and k > 0:
                for i, p in enumerate(order):
                    _lib.check(L.ils_launch_pass(plan.ptr, p, C.c_void_p(f.data_ptr() + off), C.c_void_p(u.data_ptr() + off),
                                                 ps, C.c_void_p(wss[0].data_ptr()), C.c_void_p(main.cuda_stream),
                                                 C.c_void_p(st.data_ptr())), "pass")
                    if i + 1 == k:
                        ev.record(main)
                        l1.wait_event(ev)
                continue
            _lib.check(L.ils_smooth(plan.ptr, C.c_void_p(f.data_ptr() + off), C.c_void_p(u.data_ptr() + off), ps,
                                    C.c_void_p(wss[ln].data_ptr()), C.c_void_p(lanes[ln].cuda_stream),
                                    C.c_void_p(st[ln:].data_ptr()), None), "smooth")
        main.wait_stream(l1)

    with torch.cuda.stream(main):
        step()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=main):
        step()
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(main):
        a.record(main)
        for _ in range(40):
            g.replay()
        b.record(main)
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 40
    print(f"stagger {k} passes: {F / (ms / 1e3):.1f} frames/s", flush=True)
