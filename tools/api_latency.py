"""Per-call latency of the drop-in Python API (numpy f64 in / out, the reference's
contract) on one 1080p RGB image, vs the device-resident call.

    python tools/api_latency.py
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2003_07504_b200 as ils  # noqa: E402

rng = np.random.default_rng(20240607)
planes = tuple(rng.random((1080, 1920)) for _ in range(3))
img = ils.MultiImage(planes, ils.RGB)
params = ils.SmoothParams(ils.Charbonnier(0.8, 1e-4), 1.0)
for _ in range(2):
    ils.smooth_color(img, params)
t = time.perf_counter()
n = 10
for _ in range(n):
    ils.smooth_color(img, params)
print(f"smooth_color (numpy f64 1080p RGB in/out): {(time.perf_counter() - t) / n * 1e3:.2f} ms/call")
f = torch.from_numpy(np.stack(planes)).to("cuda", torch.float32)
for _ in range(2):
    ils.smooth_batch(f, params)
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(n):
    ils.smooth_batch(f, params)
torch.cuda.synchronize()
print(f"smooth_batch (CUDA tensor in/out): {(time.perf_counter() - t) / n * 1e3:.3f} ms/call")
t = time.perf_counter()
for _ in range(n):
    ils.smooth_plane(planes[0], params)
print(f"smooth_plane (numpy f64 1080p gray): {(time.perf_counter() - t) / n * 1e3:.2f} ms/call")
