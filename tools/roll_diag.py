"""Diagnose rolling-band vs k_row differences: max |diff| and the first differing rows per case."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2003_07504_b200 as ils  # noqa: E402
from paper_2003_07504_b200 import _lib  # noqa: E402
from paper_2003_07504_b200.penalty import params_of  # noqa: E402


def run(f, params, roll, rows, iters_override=None):
    os.environ["ILS_NO_ROLL"] = "0" if roll else "1"
    os.environ["ILS_ROLL_ROWS"] = str(rows or 0)
    B, H, W = f.shape
    L = _lib.lib()
    h = C.c_void_p()
    _lib.check(L.ils_plan_create(C.byref(h), B, H, W, C.byref(params_of(params)), _lib.ILS_F32, 0))
    ws_sz = C.c_size_t()
    L.ils_workspace_size(h, C.byref(ws_sz))
    ws = torch.zeros(ws_sz.value, dtype=torch.uint8, device="cuda")
    st = torch.empty(1, dtype=torch.int32, device="cuda")
    u = torch.empty_like(f)
    _lib.check(L.ils_smooth(h, C.c_void_p(f.data_ptr()), C.c_void_p(u.data_ptr()), H * W, C.c_void_p(ws.data_ptr()),
                            C.c_void_p(torch.cuda.current_stream().cuda_stream), C.c_void_p(st.data_ptr()), None))
    torch.cuda.synchronize()
    L.ils_plan_destroy(h)
    return u


for (H, W, B, rows, it) in [(333, 3840, 2, 1, 4), (333, 3840, 2, 1, 1), (333, 3840, 1, 1, 1), (332, 3840, 1, 1, 1),
                            (333, 3840, 1, 2, 1), (333, 3840, 1, 3, 1), (64, 3840, 1, 1, 1), (64, 7680, 1, 1, 1)]:
    params = ils.SmoothParams(ils.Welsch(10 / 255), 30.0, iters=it, c=2.0)
    f = torch.from_numpy(np.random.default_rng(H + W + B).random((B, H, W))).to("cuda", torch.float32)
    a = run(f, params, True, rows)
    b = run(f, params, False, None)
    d = (a - b).abs()
    bad = torch.nonzero(d.amax(dim=2) > 0)
    print((H, W, B, rows, it), "max", float(d.max()), "rows differing", bad.shape[0], bad[:8].tolist(), flush=True)
