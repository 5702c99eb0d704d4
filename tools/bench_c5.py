"""C5 benchmark: one 7680x4320 RGB image, Welsch g=10/255, lambda=30, N=10, c=2.

    python tools/bench_c5.py                                   # 1 GPU, whole image per plane
    torchrun --nproc-per-node N tools/bench_c5.py              # N GPUs: row slabs + NCCL all-to-all

Prints one JSON line (rank 0): wall time per image (CUDA events, max over
ranks), with the slab path checked bitwise against the 1-GPU result on
rank 0's rows when N == 1 or when --check is given.
"""

import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2003_07504_b200 as ils  # noqa: E402
from paper_2003_07504_b200 import _lib, dist as D  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--h", type=int, default=4320)
ap.add_argument("--w", type=int, default=7680)
ap.add_argument("--steps", type=int, default=5)
ap.add_argument("--warmup", type=int, default=2)
ap.add_argument("--check", action="store_true")
ap.add_argument("--slab", action="store_true", help="slab + all-to-all path even on one rank")
ap.add_argument("--no-overlap", action="store_true", help="slab path plane by plane (no exchange overlap)")
a = ap.parse_args()

world = int(os.environ.get("WORLD_SIZE", "1"))
rank = int(os.environ.get("RANK", "0"))
local = int(os.environ.get("LOCAL_RANK", "0"))
torch.cuda.set_device(local)
dev = torch.device("cuda", local)
if world > 1:
    dist.init_process_group("nccl", device_id=dev)

params = ils.SmoothParams(ils.Welsch(10 / 255), 30.0, iters=10, c=2.0)
H, W = a.h, a.w
gen = torch.Generator(device=dev)
gen.manual_seed(20240607)
img = torch.rand((3, H, W), generator=gen, device=dev)  # same image on every rank

mode = "slab" if (world > 1 or a.slab) else "single"
if mode == "slab" and not dist.is_initialized():
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29544")
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
if mode == "slab":
    plan, lay = D.slab_layout(H, W, params.c_params(), _lib.ILS_F32, world, rank, device=local)
    stream = lambda: torch.cuda.current_stream(dev).cuda_stream  # noqa: E731
    alloc = lambda n: torch.zeros(n, dtype=torch.float32, device=dev)  # noqa: E731
    if a.no_overlap:
        sm = D.SlabSmoother(lay, params.iters, D.CudaSlabKernels(plan, stream), D.torch_exchange(), alloc)
    else:  # channels pipelined: one plane's all-to-all overlaps the next planes' passes
        pipe = D.SlabPipeline(lay, params.iters, D.CudaSlabKernels(plan, stream), D.torch_exchange_async(), alloc,
                              planes=3)
    rows = D.halo_rows(H, lay.row0[rank], lay.row0[rank + 1])
    f_ext = [img[c][rows].contiguous() for c in range(3)]
    u = [torch.empty((lay.rows, W), device=dev) for _ in range(3)]
    status = torch.empty(1, dtype=torch.int32, device=dev)

    def step():
        status.fill_(_lib.STATUS_CLEAN)
        if a.no_overlap:
            for c in range(3):  # plane by plane, each exchange blocking the compute stream
                sm.smooth(f_ext[c], u[c], status)
        else:
            pipe.smooth(f_ext, u, status)
else:
    def step():
        return ils.smooth_batch(img, params)

for _ in range(a.warmup):
    step()
torch.cuda.synchronize()
if dist.is_initialized():
    dist.barrier()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(a.steps):
    out = step()
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / a.steps
if dist.is_initialized():
    t = torch.tensor([ms], device=dev, dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
check = None
if a.check and mode == "slab":
    ref = ils.smooth_batch(img, params)
    r0, r1 = lay.row0[rank], lay.row0[rank + 1]
    ok = all(torch.equal(u[c], ref[c, r0:r1]) for c in range(3))
    t = torch.tensor([1 if ok else 0], device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MIN)
    check = bool(t.item())
if rank == 0:
    print(json.dumps({"metric": "C5 7680x4320 RGB ILS (Welsch, N=10) wall time per image", "value": round(ms, 3),
                      "unit": "ms", "n_gpus": world, "mode": mode + ("" if mode == "single" or a.no_overlap
                                                                     else "+overlap"), "steps": a.steps,
                      "bitwise_equal_to_1gpu": check}), flush=True)
if dist.is_initialized():
    dist.destroy_process_group()
