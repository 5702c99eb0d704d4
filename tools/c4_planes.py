"""C4 schedule experiment: 4K RGB frames smoothed per frame (3 planes per call) or per plane
(1 plane per call, the per-plane working set -- f + two half spectra, 100 MB -- fits L2), on 1 or 2 lanes.

    python tools/c4_planes.py [--frames 48]
"""
import argparse
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2003_07504_b200 as ils  # noqa: E402
from paper_2003_07504_b200 import _lib, _runtime as rt  # noqa: E402
from paper_2003_07504_b200.penalty import params_of  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--frames", type=int, default=48)
a = ap.parse_args()
H, W, CH, F = 2160, 3840, 3, a.frames
prm = ils.SmoothParams(ils.Charbonnier(0.8, 1e-4), 1.0)
f = torch.rand((F * CH, H, W), device="cuda")
u = torch.empty_like(f)
L = _lib.lib()
res = {}
for per in (3, 1):
    plan = rt.get_plan(per, H, W, params_of(prm), _lib.ILS_F32, 0)
    for nl in (1, 2, 3):
        lanes = [torch.cuda.Stream() for _ in range(nl)]
        wss = [torch.empty(plan.workspace_bytes, dtype=torch.uint8, device="cuda") for _ in lanes]
        sts = [torch.empty(1, dtype=torch.int32, device="cuda") for _ in lanes]

        def run():
            cur = torch.cuda.current_stream()
            for ln in lanes:
                ln.wait_stream(cur)
            for i in range(F * CH // per):
                k = i % nl
                off = i * per * H * W * 4
                L.ils_smooth(plan.ptr, C.c_void_p(f.data_ptr() + off), C.c_void_p(u.data_ptr() + off), H * W,
                             C.c_void_p(wss[k].data_ptr()), C.c_void_p(lanes[k].cuda_stream),
                             C.c_void_p(sts[k].data_ptr()), None)
            for ln in lanes:
                cur.wait_stream(ln)
        run()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(2):
            run()
        e1.record()
        torch.cuda.synchronize()
        res[f"planes_per_call={per} lanes={nl}"] = round(2 * F / (e0.elapsed_time(e1) / 1e3), 1)
print(json.dumps(res))
