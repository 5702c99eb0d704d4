"""Repeat one smooth_plane shape/precision against the oracle (flakiness probe).

    python tools/repro_shape.py H W prec reps
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2003_07504_b200 as ils  # noqa: E402
from oracle import ils_oracle as O  # noqa: E402

H, W, prec, reps = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3], int(sys.argv[4])
f = np.random.default_rng(5).random((H, W))
params = ils.SmoothParams(ils.Charbonnier(0.8, 1e-4), 1.0, iters=4)
ref = O.smooth_plane(f, O.Charbonnier(0.8, 1e-4), 1.0, 4)
for i in range(reps):
    u = ils.smooth_plane(f, params, precision=prec)
    err = np.max(np.abs(u - ref))
    bad = np.argwhere(np.abs(u - ref) > 1e-6)
    print(f"{H}x{W} {prec} rep {i}: max-abs {err:.3e}, bad px {len(bad)}", bad[:4].tolist() if len(bad) else "",
          flush=True)
