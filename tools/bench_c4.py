"""C4 benchmark: 3840x2160 RGB video, 256 frames, Charbonnier p=0.8, lambda=1, N=4.

    python tools/bench_c4.py                          # 1 GPU
    torchrun --nproc-per-node N tools/bench_c4.py     # frames sharded over N GPUs, no communication

Frame k is generated on the device from seed 20240607 + k, so
every rank can produce its own shard and the per-frame result does not
depend on the rank count.  Prints one JSON line (rank 0): aggregate frames/s
= frames / max-over-ranks device time, plus a per-frame checksum so runs at
different N can be compared bit for bit.
"""

import argparse
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2003_07504_b200 as ils  # noqa: E402
from paper_2003_07504_b200 import _lib, _runtime as rt, dist as D  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--frames", type=int, default=256)
ap.add_argument("--h", type=int, default=2160)
ap.add_argument("--w", type=int, default=3840)
ap.add_argument("--lanes", type=int, default=2)
ap.add_argument("--reps", type=int, default=2)
a = ap.parse_args()

world = int(os.environ.get("WORLD_SIZE", "1"))
rank = int(os.environ.get("RANK", "0"))
local = int(os.environ.get("LOCAL_RANK", "0"))
torch.cuda.set_device(local)
dev = torch.device("cuda", local)
if world > 1:
    dist.init_process_group("nccl", device_id=dev)
H, W, CH = a.h, a.w, 3
mine = D.frame_shard(a.frames, world, rank)
prm = ils.SmoothParams(ils.Charbonnier(0.8, 1e-4), 1.0)
plan = rt.get_plan(CH, H, W, prm.c_params(), _lib.ILS_F32, local)
L = _lib.lib()
frames = torch.empty((len(mine), CH, H, W), device=dev)
for i, k in enumerate(mine):
    g = torch.Generator(device=dev)
    g.manual_seed(20240607 + k)
    frames[i] = torch.rand((CH, H, W), generator=g, device=dev)
out = torch.empty_like(frames)
lanes = [torch.cuda.Stream(device=dev) for _ in range(a.lanes)]
wss = [torch.empty(plan.workspace_bytes, dtype=torch.uint8, device=dev) for _ in lanes]
sts = [torch.full((1,), _lib.STATUS_CLEAN, dtype=torch.int32, device=dev) for _ in lanes]


def run_all():
    cur = torch.cuda.current_stream(dev)
    for ln in lanes:
        ln.wait_stream(cur)
    for i in range(len(mine)):
        k = i % len(lanes)
        _lib.check(L.ils_smooth(plan.ptr, C.c_void_p(frames[i].data_ptr()), C.c_void_p(out[i].data_ptr()), H * W,
                                C.c_void_p(wss[k].data_ptr()), C.c_void_p(lanes[k].cuda_stream),
                                C.c_void_p(sts[k].data_ptr()), None), "ils_smooth")
    for ln in lanes:
        cur.wait_stream(ln)


run_all()
torch.cuda.synchronize()
for s in sts:
    rt.raise_status(int(s.item()))
if world > 1:
    dist.barrier()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(a.reps):
    run_all()
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / a.reps
if world > 1:
    t = torch.tensor([ms], device=dev, dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
# per-frame checksums (sum of squares in f64) gathered to rank 0 in frame order
cs = (out.double() ** 2).sum(dim=(1, 2, 3)).cpu().tolist()
allcs = [None] * world
if world > 1:
    dist.all_gather_object(allcs, cs)
else:
    allcs = [cs]
if rank == 0:
    flat = [x for part in allcs for x in part]
    print(json.dumps({"metric": "C4 3840x2160 RGB video ILS (N=4), aggregate frames/s", "value": round(a.frames / (ms / 1e3), 2),
                      "unit": "frames/s", "n_gpus": world, "frames": a.frames, "ms_total": round(ms, 3),
                      "lanes": a.lanes, "checksum_first": flat[0], "checksum_sum": sum(flat)}), flush=True)
if world > 1:
    dist.destroy_process_group()
