"""Where the numpy drop-in's time goes (smooth_color on float64 planes, 1080p RGB):
host staging, H2D, compute, D2H + widening -- and alternatives for each."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2003_07504_b200 as ils  # noqa: E402
from paper_2003_07504_b200 import _runtime as rt  # noqa: E402

H, W = 1080, 1920
rng = np.random.default_rng(1)
planes = [rng.random((H, W)) for _ in range(3)]
img = ils.MultiImage(tuple(planes), ils.RGB)
params = ils.SmoothParams(ils.Charbonnier(0.8, 1e-4), 1.0)


def t(fn, n=10):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        r = fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / n * 1e3, r


res = {}
res["smooth_color_ms"], _ = t(lambda: ils.smooth_color(img, params))
res["to_device_planes_ms"], dev = t(lambda: rt.to_device_planes(planes))
res["smooth_device_ms"], (u, _, _) = t(lambda: rt.smooth_device(dev, params.c_params()))
res["to_host_f64_ms"], _ = t(lambda: rt.to_host_f64(u))
stage = torch.empty((3, H, W), dtype=torch.float64, pin_memory=True)
res["host_copy_into_pinned_ms"], _ = t(lambda: [np.copyto(stage.numpy()[i], planes[i]) for i in range(3)])
res["h2d_pinned_f64_ms"], _ = t(lambda: stage.to("cuda", non_blocking=True))
res["h2d_pageable_f64_ms"], _ = t(lambda: [torch.from_numpy(p).to("cuda") for p in planes])
d64 = torch.empty((3, H, W), dtype=torch.float64, device="cuda")
res["d2h_f64_into_fresh_pinned_ms"], _ = t(lambda: d64.to("cpu", non_blocking=False).pin_memory())
res["d2h_f64_into_torch_pinned_empty_ms"], _ = t(
    lambda: torch.empty((3, H, W), dtype=torch.float64, pin_memory=True).copy_(d64, non_blocking=True))
res["d2h_f64_pageable_ms"], _ = t(lambda: d64.cpu())
res["np_empty_plus_copy_ms"], _ = t(lambda: [np.copyto(np.empty((H, W)), planes[i]) for i in range(3)])
print({k: round(v, 3) for k, v in res.items()})

# input alternatives: pageable H2D of each plane from its own thread / stream
from concurrent.futures import ThreadPoolExecutor  # noqa: E402

pool = ThreadPoolExecutor(3)
streams = [torch.cuda.Stream() for _ in range(3)]
dst = torch.empty((3, H, W), dtype=torch.float64, device="cuda")


def par_pageable():
    def one(i):
        with torch.cuda.stream(streams[i]):
            dst[i].copy_(torch.from_numpy(planes[i]), non_blocking=True)
            streams[i].synchronize()
    list(pool.map(one, range(3)))


res2 = {}
res2["h2d_pageable_3threads_ms"], _ = t(par_pageable)
stage3 = [torch.empty((H, W), dtype=torch.float64, pin_memory=True) for _ in range(3)]


def par_staged():
    def one(i):
        np.copyto(stage3[i].numpy(), planes[i])
        with torch.cuda.stream(streams[i]):
            dst[i].copy_(stage3[i], non_blocking=True)
            streams[i].synchronize()
    list(pool.map(one, range(3)))


res2["staged_per_plane_3threads_ms"], _ = t(par_staged)
print({k: round(v, 3) for k, v in res2.items()})
