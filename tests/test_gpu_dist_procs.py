"""C5 slab decomposition across real processes, with the real CUDA passes (needs a GPU).

Two (and three) OS processes -- one rank each, gloo process group -- run
dist.SlabSmoother with the CUDA slab kernels (ils_slab_row_pass /
ils_slab_col_pass) on cuda:0.  The transposes go through gloo's
all_to_all_single on CPU-staged copies of the device blocks (the host
waits for each rank's kernels before its exchange, so no kernel ever waits
on another process).  Every rank's rows must be bit-identical to the
single-GPU smooth of the whole image ("P-GPU output can be
bit-identical to the 1-GPU output").  The NCCL exchange itself is covered by
tests/test_gpu_parity.py::test_slab_pipeline_nccl_one_rank_bitwise and the
bench's c5 leg at N > 1.
"""

import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs CUDA")]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _staged_exchange():
    """all_to_all over gloo: device send block -> host, exchange, host -> device recv block."""
    import torch.distributed as dist

    def run(send, recv, send_counts, recv_counts):
        torch.cuda.current_stream().synchronize()  # this rank's producing pass is done
        hs, hr = send.cpu(), torch.empty(recv.numel(), dtype=recv.dtype)
        dist.all_to_all_single(hr, hs, recv_counts, send_counts)
        recv.copy_(hr)

    return run


def _worker(rank, world, port, H, W, kind, q):
    import torch.distributed as dist

    import paper_2003_07504_b200 as ils
    from paper_2003_07504_b200 import _lib
    from paper_2003_07504_b200 import dist as D
    from paper_2003_07504_b200.penalty import params_of

    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        params = (ils.SmoothParams(ils.Charbonnier(0.8, 1e-4), 1.0, iters=4) if kind == 0 else
                  ils.SmoothParams(ils.Welsch(10 / 255), 30.0, iters=5, c=2.0))
        img = torch.from_numpy(np.random.default_rng(77).random((H, W))).to("cuda", torch.float32)
        plan, lay = D.slab_layout(H, W, params_of(params), _lib.ILS_F32, world, rank, device=0)
        stream = lambda: torch.cuda.current_stream().cuda_stream  # noqa: E731
        alloc = lambda n: torch.zeros(n, dtype=torch.float32, device="cuda")  # noqa: E731
        sm = D.SlabSmoother(lay, params.iters, D.CudaSlabKernels(plan, stream), _staged_exchange(), alloc)
        r0, r1 = lay.row0[rank], lay.row0[rank + 1]
        f_ext = img[D.halo_rows(H, r0, r1)].contiguous()
        u = torch.empty((r1 - r0, W), device="cuda")
        status = torch.full((1,), _lib.STATUS_CLEAN, dtype=torch.int32, device="cuda")
        sm.smooth(f_ext, u, status)
        torch.cuda.synchronize()
        ref = ils.smooth_batch(img[None], params)[0]
        ok = int(status.item()) == _lib.STATUS_CLEAN and torch.equal(u, ref[r0:r1])
        _lib.lib().ils_plan_destroy(plan)
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, bool(ok), ""))
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, False, repr(e)))


@pytest.mark.parametrize("world,H,W,kind", [(2, 360, 640, 0), (2, 1080, 1920, 1), (3, 270, 480, 0)])
def test_slab_processes_bitwise_equal_single_gpu(world, H, W, kind):
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, H, W, kind, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    assert all(ok for _, ok, _ in res), res


@pytest.mark.parametrize("H,W,planes", [(360, 640, 3), (1080, 1920, 1), (4320, 7680, 1)])
def test_smooth_dist_c_entry_nccl_one_rank_bitwise(H, W, planes):
    # ils_smooth_dist (C ABI: slab passes + NCCL send/recv issued from C) on a
    # 1-rank communicator the library creates: bitwise the 1-GPU ils_smooth
    import paper_2003_07504_b200 as ils
    from paper_2003_07504_b200 import _lib
    from paper_2003_07504_b200 import dist as D

    params = ils.SmoothParams(ils.Welsch(10 / 255), 30.0, iters=3, c=2.0)
    img = torch.from_numpy(np.random.default_rng(H).random((planes, H, W))).to("cuda", torch.float32)
    ns = D.NcclSlab(H, W, params, 1, 0, device=0)
    try:
        rows = D.halo_rows(H, 0, H)
        f_ext = img[:, rows].contiguous()
        u = torch.empty((planes, H, W), device="cuda")
        ns.smooth(f_ext, u)
        torch.cuda.synchronize()
        assert int(ns.status.item()) == _lib.STATUS_CLEAN
        ref = ils.smooth_batch(img, params)
        assert torch.equal(u, ref)
    finally:
        ns.close()


def test_smooth_dist_rejects_non_slab_plans_and_bad_strides():
    import ctypes as C

    import paper_2003_07504_b200 as ils
    from paper_2003_07504_b200 import _lib, _runtime as rt
    from paper_2003_07504_b200 import dist as D

    params = ils.SmoothParams(ils.Charbonnier(0.8, 1e-4), 1.0)
    plan = rt.get_plan(1, 64, 64, params.c_params(), _lib.ILS_F32, 0)
    L = _lib.lib()
    buf = torch.empty(1 << 16, device="cuda")
    rc = L.ils_smooth_dist(plan.ptr, C.c_void_p(buf.data_ptr()), C.c_void_p(buf.data_ptr()), 1, 66 * 64, 64 * 64,
                           C.c_void_p(buf.data_ptr()), C.c_void_p(1), None, C.c_void_p(buf.data_ptr()))
    assert rc == _lib.ILS_EINVAL and "slab" in _lib.last_error()
    ns = D.NcclSlab(64, 64, params, 1, 0, device=0)
    try:
        rc = L.ils_smooth_dist(ns.plan, C.c_void_p(buf.data_ptr()), C.c_void_p(buf.data_ptr()), 1, 64 * 64, 64 * 64,
                               C.c_void_p(ns.ws.data_ptr()), ns.comm, None, C.c_void_p(ns.status.data_ptr()))
        assert rc == _lib.ILS_EINVAL  # f_ext must hold the rows plus two halo rows
    finally:
        ns.close()
