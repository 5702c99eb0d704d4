"""Working-set probe: 32 1080p RGB frames per step as calls of P planes over S
graph lanes (P=3, S=2 is the bench); smaller P shrinks each lane's L2 working set."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2003_07504_b200 as ils  # noqa: E402
from paper_2003_07504_b200 import _lib, _runtime as rt  # noqa: E402

H, W, F, CH = 1080, 1920, 32, 3
params = ils.SmoothParams(ils.Charbonnier(0.8, 1e-4), 1.0)
f = torch.rand((F * CH, H, W), device="cuda")
u = torch.empty_like(f)
L = _lib.lib()
for P, S in [(3, 2), (3, 1), (1, 2), (1, 3), (1, 4), (1, 6), (3, 3)]:
    plan = rt.get_plan(P, H, W, params.c_params(), _lib.ILS_F32, 0)
    wss = [torch.empty(plan.workspace_bytes, dtype=torch.uint8, device="cuda") for _ in range(S)]
    st = torch.empty(S, dtype=torch.int32, device="cuda")
    main = torch.cuda.Stream()
    lanes = [main] + [torch.cuda.Stream() for _ in range(S - 1)]

    def step():
        for ln in lanes[1:]:
            ln.wait_stream(main)
        for gi, p0 in enumerate(range(0, F * CH, P)):
            k = gi % S
            _lib.check(L.ils_smooth(plan.ptr, C.c_void_p(f[p0].data_ptr()), C.c_void_p(u[p0].data_ptr()), H * W,
                                    C.c_void_p(wss[k].data_ptr()), C.c_void_p(lanes[k].cuda_stream),
                                    C.c_void_p(st[k:].data_ptr()), None), "smooth")
        for ln in lanes[1:]:
            main.wait_stream(ln)

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
        for _ in range(30):
            g.replay()
        b.record(main)
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 30
    print(f"P={P} S={S}: {F / (ms / 1e3):.1f} frames/s")
