"""Where the numpy drop-in's time goes (smooth_color on float64 planes, 1080p RGB):
chunked pinned staging in, compute, pooled pinned results out -- per staging
chunk size, and the host-side alternatives (pageable copies, fresh arrays)."""
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


def t(fn, n=20):
    r = fn()
    torch.cuda.synchronize()
    del r
    t0 = time.perf_counter()
    for _ in range(n):
        r = fn()
        del r
    torch.cuda.synchronize()
    return round((time.perf_counter() - t0) / n * 1e3, 3)


print("host threads", rt._HOST_THREADS, "cpus", os.cpu_count())
for chunk in (1 << 20, 2 << 20, 4 << 20, 8 << 20, 1 << 30):
    rt._CHUNK_BYTES = chunk
    dev = rt.to_device_planes(planes)
    u, _, _ = rt.smooth_device(dev, params.c_params())
    print({"chunk_MB": chunk / 2**20, "smooth_color_ms": t(lambda: ils.smooth_color(img, params)),
           "to_device_planes_ms": t(lambda: rt.to_device_planes(planes)),
           "smooth_device_ms": t(lambda: rt.smooth_device(dev, params.c_params())),
           "to_host_f64_pooled_ms": t(lambda: rt.to_host_f64(u))})
rt._CHUNK_BYTES = 4 << 20
rt._HOST_NARROW = True
for chunk in (2 << 20, 4 << 20):
    rt._CHUNK_BYTES = chunk
    print({"host_narrow_chunk_MB": chunk / 2**20, "smooth_color_ms": t(lambda: ils.smooth_color(img, params)),
           "to_device_planes_ms": t(lambda: rt.to_device_planes(planes))})
rt._HOST_NARROW = False
rt._CHUNK_BYTES = 4 << 20
lim, pool = rt._OUT_LIMIT, rt._out_pool
rt._OUT_LIMIT, rt._out_pool = 0, rt._OutPool()
print({"to_host_f64_plain_ms": t(lambda: rt.to_host_f64(u)),
       "smooth_color_plain_out_ms": t(lambda: ils.smooth_color(img, params))})
rt._OUT_LIMIT, rt._out_pool = lim, pool
d64 = torch.empty((3, H, W), dtype=torch.float64, device="cuda")
pin = torch.empty((3, H, W), dtype=torch.float64, pin_memory=True)
print({"h2d_pinned_f64_ms": t(lambda: pin.to("cuda", non_blocking=True)),
       "d2h_pinned_f64_ms": t(lambda: pin.copy_(d64, non_blocking=True)),
       "h2d_pageable_f64_ms": t(lambda: [torch.from_numpy(p).to("cuda") for p in planes]),
       "np_empty_plus_copy_ms": t(lambda: [np.copyto(np.empty((H, W)), planes[i]) for i in range(3)]),
       "host_copy_into_pinned_1thread_ms": t(lambda: [np.copyto(pin.numpy()[i], planes[i]) for i in range(3)])})
