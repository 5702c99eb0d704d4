"""Time each pass of the 1080p RGB plan alone (CUDA events), for tuning sweeps.

    ILS_ROW_BAND=8 python tools/time_passes.py [--planes 3]
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

ap = argparse.ArgumentParser()
ap.add_argument("--planes", type=int, default=3)
ap.add_argument("--h", type=int, default=1080)
ap.add_argument("--w", type=int, default=1920)
ap.add_argument("--reps", type=int, default=50)
a = ap.parse_args()
params = ils.SmoothParams(ils.Charbonnier(0.8, 1e-4), 1.0)
f = torch.rand((a.planes, a.h, a.w), device="cuda")
u = torch.empty_like(f)
plan = rt.get_plan(a.planes, a.h, a.w, params.c_params(), _lib.ILS_F32, 0)
ws = torch.empty(plan.workspace_bytes, dtype=torch.uint8, device="cuda")
st = torch.empty(1, dtype=torch.int32, device="cuda")
L = _lib.lib()
s = torch.cuda.current_stream()
out = {"env": {k: v for k, v in os.environ.items() if k.startswith("ILS_")},
       "plan": {k: plan.info[k] for k in ("row_band", "row_grid", "col_cols", "col_grid")}}
for p, name in ((0, "row_f0"), (1, "col"), (2, "row_it"), (3, "row_fin")):
    def launch():
        _lib.check(L.ils_launch_pass(plan.ptr, p, C.c_void_p(f.data_ptr()), C.c_void_p(u.data_ptr()), a.h * a.w,
                                     C.c_void_p(ws.data_ptr()), C.c_void_p(s.cuda_stream),
                                     C.c_void_p(st.data_ptr())), "pass")
    for _ in range(5):
        launch()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(a.reps):
        launch()
    e1.record(s)
    torch.cuda.synchronize()
    out[name] = round(e0.elapsed_time(e1) / a.reps * 1e3, 2)
print(json.dumps(out))
