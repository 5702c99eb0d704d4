"""Multi-GPU drivers: frame sharding (C4) and slab FFT (C5).

One process per GPU, torch.distributed for the plumbing (NCCL on GPUs, gloo
in the CPU tests).

C4 -- video batches: frames are independent; rank r smooths frames
      frame_shard(F, P, r) with no communication.  A plane's result is
      bitwise independent of where it is computed, so the
      sharded output equals the 1-GPU output.
C5 -- one large image: rank r owns a row slab for the row passes and a
      column slab of the half spectrum for the column passes.  Per
      iteration the spectrum crosses the ranks twice with an all-to-all
      (row -> column, then column -> row with the +-1 halo rows folded in),
      which is the only exchange step of the algorithm.  The CUDA kernels
      read and write the all-to-all blocks directly (include/ils_b200.h,
      ils_slab_*), so there is no separate pack/unpack pass.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

from . import _lib
from .penalty import params_of

_MAXSEG = 8


def frame_shard(n_frames: int, world: int, rank: int) -> range:
    """Contiguous, balanced frame range of `rank` (C4, weak or strong scaling)."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError(f"bad rank {rank} of {world}")
    lo = n_frames * rank // world
    hi = n_frames * (rank + 1) // world
    return range(lo, hi)


def smooth_frames_sharded(frames, params, group=None):
    """C4: smooth this rank's frames [F_local, C, H, W] (CUDA tensor) in one launch sequence."""
    from .smoother import smooth_batch

    f = frames.reshape(-1, frames.shape[-2], frames.shape[-1])
    return smooth_batch(f, params).reshape(frames.shape)


@dataclass
class SlabLayout:
    """Row / column split of one H x W image over P ranks (from the C planner)."""

    P: int
    rank: int
    height: int
    width: int
    row0: list
    col0: list
    pitch: list
    counts: list  # [fwd_send, fwd_recv, rev_send, rev_recv] per peer, complex elements

    @property
    def rows(self):
        return self.row0[self.rank + 1] - self.row0[self.rank]

    @property
    def cols(self):
        return self.col0[self.rank + 1] - self.col0[self.rank]

    def size(self, which: int) -> int:
        return sum(self.counts[which])


def slab_layout(height, width, cparams, dtype_code, nranks, rank, device=-1):
    """Plan (device >= 0) or host-only layout (device = -1) of a slab decomposition."""
    L = _lib.lib()
    h = C.c_void_p()
    _lib.check(L.ils_slab_plan_create(C.byref(h), height, width, C.byref(cparams), dtype_code, device, nranks, rank),
               "ils_slab_plan_create")
    row0 = (C.c_int32 * (_MAXSEG + 1))()
    col0 = (C.c_int32 * (_MAXSEG + 1))()
    pitch = (C.c_int32 * _MAXSEG)()
    counts = (C.c_int64 * (4 * _MAXSEG))()
    _lib.check(L.ils_slab_get_layout(h, row0, col0, pitch, counts), "ils_slab_get_layout")
    lay = SlabLayout(nranks, rank, height, width, list(row0[: nranks + 1]), list(col0[: nranks + 1]),
                     list(pitch[:nranks]), [list(counts[k * _MAXSEG: k * _MAXSEG + nranks]) for k in range(4)])
    return h, lay


def halo_rows(height: int, r0: int, r1: int):
    """Global row indices of a slab's rows plus its periodic halo rows."""
    return [(r0 - 1) % height] + list(range(r0, r1)) + [r1 % height]


class CudaSlabKernels:
    """The CUDA row/column passes of one rank (ils_slab_row_pass / ils_slab_col_pass)."""

    def __init__(self, plan_ptr, stream_fn):
        self.plan = plan_ptr
        self.stream_fn = stream_fn
        self.L = _lib.lib()

    def row(self, mode, f_ext, rev_recv, fwd_send, u, it, status):
        p = lambda t: C.c_void_p(t.data_ptr()) if t is not None else None  # noqa: E731
        _lib.check(self.L.ils_slab_row_pass(self.plan, mode, p(f_ext), p(rev_recv), p(fwd_send), p(u), it,
                                            C.c_void_p(self.stream_fn()), p(status)), "ils_slab_row_pass")

    def col(self, fwd_recv, rev_send):
        _lib.check(self.L.ils_slab_col_pass(self.plan, C.c_void_p(fwd_recv.data_ptr()),
                                            C.c_void_p(rev_send.data_ptr()), C.c_void_p(self.stream_fn())),
                   "ils_slab_col_pass")


def torch_exchange(group=None):
    """all-to-all of flat real views (NCCL on CUDA tensors, gloo on CPU)."""
    import torch.distributed as dist

    def run(send, recv, send_counts, recv_counts):
        dist.all_to_all_single(recv, send, recv_counts, send_counts, group=group)

    return run


class SlabSmoother:
    """C5: ILS on one image whose rows are sharded over the ranks of a group.

    smooth(f_ext) takes this rank's rows plus the two periodic halo rows
    ([rows + 2, W]) and returns its rows of u.  `kernels` and `exchange` are
    injectable so the same driver runs on GPUs (CUDA passes + NCCL) and in
    the CPU tests (reference-math passes + gloo).
    """

    def __init__(self, layout: SlabLayout, iters: int, kernels, exchange, alloc, real_per_complex=2):
        self.lay = layout
        self.iters = iters
        self.k = kernels
        self.x = exchange
        rpc = real_per_complex
        self.rpc = rpc
        c = layout.counts
        self.fwd_send = alloc(rpc * layout.size(0))
        self.fwd_recv = alloc(rpc * layout.size(1))
        self.rev_send = alloc(rpc * layout.size(2))
        self.rev_recv = alloc(rpc * layout.size(3))
        self.fwd_sc = [rpc * n for n in c[0]]
        self.fwd_rc = [rpc * n for n in c[1]]
        self.rev_sc = [rpc * n for n in c[2]]
        self.rev_rc = [rpc * n for n in c[3]]

    def smooth(self, f_ext, u, status):
        """All iterations; `status` is the device status word (ILS_STATUS_CLEAN when fine)."""
        k, x = self.k, self.x
        k.row(0, f_ext, None, self.fwd_send, None, 0, status)
        for n in range(self.iters):
            x(self.fwd_send, self.fwd_recv, self.fwd_sc, self.fwd_rc)
            k.col(self.fwd_recv, self.rev_send)
            x(self.rev_send, self.rev_recv, self.rev_sc, self.rev_rc)
            if n + 1 < self.iters:
                k.row(1, f_ext, self.rev_recv, self.fwd_send, None, n + 1, status)
        k.row(3, f_ext, self.rev_recv, None, u, self.iters, status)
        return u


def torch_exchange_async(group=None):
    """Non-blocking all-to-all: returns the work handle (NCCL: `wait()` makes the
    current CUDA stream wait for the exchange, the host does not block)."""
    import torch.distributed as dist

    def run(send, recv, send_counts, recv_counts):
        return dist.all_to_all_single(recv, send, recv_counts, send_counts, group=group, async_op=True)

    return run


class SlabPipeline:
    """C5 with the exchanges overlapped: the planes (colour channels) of one image
    move through the slab passes as a software pipeline ("pipeline
    the 3 channels").  While plane c's all-to-all is in flight -- NCCL runs it
    on its own stream, `async_op=True` -- the next planes' row or column passes
    run on the compute stream; plane c's next pass waits only for its own
    exchange (`work.wait()` orders the compute stream after it).  Each plane has
    its own send/receive buffers; the kernels and the exchange blocks are the
    SlabSmoother's, so every plane's result is bit-identical to it.
    """

    def __init__(self, layout: SlabLayout, iters: int, kernels, exchange_async, alloc, planes=3,
                 real_per_complex=2):
        self.lay, self.iters, self.k, self.x = layout, iters, kernels, exchange_async
        self.planes = [SlabSmoother(layout, iters, kernels, None, alloc, real_per_complex) for _ in range(planes)]

    def _fwd(self, s):
        return self.x(s.fwd_send, s.fwd_recv, s.fwd_sc, s.fwd_rc)

    def _rev(self, s):
        return self.x(s.rev_send, s.rev_recv, s.rev_sc, s.rev_rc)

    def smooth(self, f_exts, us, status):
        k, P = self.k, self.planes
        pend = []
        for c, s in enumerate(P):
            k.row(0, f_exts[c], None, s.fwd_send, None, 0, status)
            pend.append(self._fwd(s))  # plane c's transpose overlaps plane c+1's row pass
        for n in range(self.iters):
            for c, s in enumerate(P):
                pend[c].wait()
                k.col(s.fwd_recv, s.rev_send)
                pend[c] = self._rev(s)
            for c, s in enumerate(P):
                pend[c].wait()
                if n + 1 < self.iters:
                    k.row(1, f_exts[c], s.rev_recv, s.fwd_send, None, n + 1, status)
                    pend[c] = self._fwd(s)
                else:
                    k.row(3, f_exts[c], s.rev_recv, None, us[c], self.iters, status)
        return us


class EmulatedSlab:
    """All P ranks of a slab decomposition on ONE GPU, in lockstep.

    The per-rank CUDA passes are the real ones; the all-to-all is emulated
    by device copies between the ranks' buffers (same blocks, same order as
    NCCL's all_to_all_single).  Used by the tests to check the C5 kernels
    bitwise against the 1-GPU path without waiting kernels or extra GPUs.
    """

    def __init__(self, height, width, params, nranks, device=0, dtype_code=_lib.ILS_F32):
        import torch

        self.torch = torch
        self.P = nranks
        self.params = params
        cp = params_of(params)
        self.plans, self.lays = [], []
        for r in range(nranks):
            h, lay = slab_layout(height, width, cp, dtype_code, nranks, r, device=device)
            self.plans.append(h)
            self.lays.append(lay)
        real = torch.float32 if dtype_code == _lib.ILS_F32 else torch.float64
        dev = torch.device("cuda", device)
        alloc = lambda n: torch.zeros(n, dtype=real, device=dev)  # noqa: E731
        stream = lambda: torch.cuda.current_stream(dev).cuda_stream  # noqa: E731
        self.ranks = [SlabSmoother(lay, params.iters, CudaSlabKernels(h, stream), None, alloc)
                      for h, lay in zip(self.plans, self.lays)]
        self.real, self.dev = real, dev

    def _a2a(self, which_send, which_recv, ci_send, ci_recv):
        P = self.P
        for r in range(P):
            src = getattr(self.ranks[r], which_send)
            soff = 0
            for q in range(P):
                n = 2 * self.lays[r].counts[ci_send][q]
                dst = getattr(self.ranks[q], which_recv)
                doff = sum(2 * self.lays[q].counts[ci_recv][rr] for rr in range(r))
                dst[doff: doff + n].copy_(src[soff: soff + n])
                soff += n

    def smooth(self, f):
        """f: CUDA tensor [H, W] -> u [H, W] through P emulated ranks."""
        torch = self.torch
        H, W = f.shape
        status = torch.empty(1, dtype=torch.int32, device=self.dev)
        status.fill_(_lib.STATUS_CLEAN)
        f_ext, us = [], []
        for lay in self.lays:
            rows = halo_rows(H, lay.row0[lay.rank], lay.row0[lay.rank + 1])
            f_ext.append(f[rows].contiguous())
            us.append(torch.empty((lay.rows, W), dtype=f.dtype, device=self.dev))
        iters = self.params.iters
        for r, rk in enumerate(self.ranks):
            rk.k.row(0, f_ext[r], None, rk.fwd_send, None, 0, status)
        for n in range(iters):
            self._a2a("fwd_send", "fwd_recv", 0, 1)
            for rk in self.ranks:
                rk.k.col(rk.fwd_recv, rk.rev_send)
            self._a2a("rev_send", "rev_recv", 2, 3)
            for r, rk in enumerate(self.ranks):
                if n + 1 < iters:
                    rk.k.row(1, f_ext[r], rk.rev_recv, rk.fwd_send, None, n + 1, status)
                else:
                    rk.k.row(3, f_ext[r], rk.rev_recv, None, us[r], iters, status)
        s = int(status.item())
        from ._runtime import raise_status

        raise_status(s)
        return torch.cat(us)

    def __del__(self):
        try:
            for h in self.plans:
                _lib.lib().ils_plan_destroy(h)
        except Exception:
            pass


class NcclSlab:
    """C5 through the library's own C entry point (ils_smooth_dist): the slab
    passes with the transposes as NCCL send/recv issued from C, on one
    NCCL communicator the library creates (ils_nccl_comm_create) -- the
    unique id travels over the caller's torch.distributed group (any
    backend), or nothing when nranks == 1.
    """

    def __init__(self, height, width, params, nranks, rank, device=0, group=None, dtype_code=_lib.ILS_F32):
        import torch

        self.torch = torch
        self.plan, self.lay = slab_layout(height, width, params_of(params), dtype_code, nranks, rank, device=device)
        L = _lib.lib()
        nid = _lib.NcclId()
        if rank == 0:
            _lib.check(L.ils_nccl_get_unique_id(C.byref(nid)), "ils_nccl_get_unique_id")
        if nranks > 1:
            import torch.distributed as dist

            box = [bytes(nid.internal) if rank == 0 else None]
            dist.broadcast_object_list(box, src=0, group=group)
            C.memmove(C.addressof(nid), box[0], 128)
        self.comm = C.c_void_p()
        _lib.check(L.ils_nccl_comm_create(C.byref(self.comm), nranks, C.byref(nid), rank, device),
                   "ils_nccl_comm_create")
        ws = C.c_size_t()
        _lib.check(L.ils_dist_workspace_size(self.plan, C.byref(ws)), "ils_dist_workspace_size")
        self.ws = torch.empty(ws.value, dtype=torch.uint8, device=torch.device("cuda", device))
        self.status = torch.empty(1, dtype=torch.int32, device=torch.device("cuda", device))
        self.W = width

    def smooth(self, f_ext, u):
        """f_ext: [planes, rows + 2, W] (halo rows included), u: [planes, rows, W], CUDA, contiguous."""
        torch = self.torch
        P = f_ext.shape[0]
        _lib.check(_lib.lib().ils_smooth_dist(self.plan, C.c_void_p(f_ext.data_ptr()), C.c_void_p(u.data_ptr()), P,
                                              f_ext[0].numel(), u[0].numel(), C.c_void_p(self.ws.data_ptr()),
                                              self.comm, C.c_void_p(torch.cuda.current_stream().cuda_stream),
                                              C.c_void_p(self.status.data_ptr())), "ils_smooth_dist")
        return u

    def close(self):
        if getattr(self, "comm", None):
            _lib.lib().ils_nccl_comm_destroy(self.comm)
            self.comm = None
        if getattr(self, "plan", None):
            _lib.lib().ils_plan_destroy(self.plan)
            self.plan = None
