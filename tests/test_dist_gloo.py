"""Multi-rank host logic on CPU (gloo, world_size 2 and 3).

The C5 slab driver (paper_2003_07504_b200.dist.SlabSmoother) runs for real:
the C planner's row/column split and all-to-all counts (host-only slab
plans, no GPU), the exchange over gloo all_to_all_single, the halo rows the
reverse transpose delivers.  Only the per-rank passes are swapped for a
reference-math backend (numpy FFTs on exactly the blocks the CUDA passes
read and write), so a layout, count or halo mistake shows up as a mismatch
against the oracle's single-image smooth_plane.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2003_07504_b200 import _lib
from paper_2003_07504_b200 import dist as D
from paper_2003_07504_b200.smoother import SmoothParams
from paper_2003_07504_b200.penalty import Charbonnier, Welsch


class RefSlabKernels:
    """numpy stand-in for ils_slab_row_pass / ils_slab_col_pass (same buffer layouts, f64)."""

    def __init__(self, lay: D.SlabLayout, pen, lam, c):
        self.lay, self.pen, self.lam, self.c = lay, pen, lam, c
        self.Wc = lay.width // 2 + 1

    def _blocks(self, flat, rows_of, pitch_of, n):
        """Split a flat real buffer into complex blocks [rows_of(q)][pitch_of(q)]."""
        z = flat.numpy().view(np.complex128)
        out, off = [], 0
        for q in range(n):
            sz = rows_of(q) * pitch_of(q)
            out.append(z[off: off + sz].reshape(rows_of(q), pitch_of(q)))
            off += sz
        return out

    def _aux(self, x):
        return self.c * x - self.pen.derivative(x)

    def row(self, mode, f_ext, rev_recv, fwd_send, u, it, status):
        lay, W, P = self.lay, self.lay.width, self.lay.P
        rows = lay.rows
        fe = f_ext.numpy()
        if mode == 0:
            ue = fe.copy()
        else:
            blocks = self._blocks(rev_recv, lambda q: rows + 2, lambda q: lay.pitch[q], P)
            Y = np.concatenate([blocks[q][:, : lay.col0[q + 1] - lay.col0[q]] for q in range(P)], axis=1)
            ue = np.fft.irfft(Y * W, n=W, axis=1)
        if not np.all(np.isfinite(ue[1:-1])):
            status[0] = min(int(status[0]), 0 if mode == 0 else it)
        if mode == 3:
            u.numpy()[:] = ue[1:-1]
            return
        mx = self._aux(np.roll(ue, -1, axis=1) - ue)
        my = self._aux(ue[1:] - ue[:-1])  # my[r] = aux(u[r+1] - u[r]) for ext rows
        a = np.roll(mx, 1, axis=1)[1:-1] - mx[1:-1] + my[:-1] - my[1:]
        rhs = fe[1:-1] + self.lam / 2.0 * a
        R = np.fft.rfft(rhs, axis=1)
        out = self._blocks(fwd_send, lambda q: rows, lambda q: lay.pitch[q], P)
        for q in range(P):
            out[q][:, : lay.col0[q + 1] - lay.col0[q]] = R[:, lay.col0[q]: lay.col0[q + 1]]

    def col(self, fwd_recv, rev_send):
        lay, H, W, me = self.lay, self.lay.height, self.lay.width, self.lay.rank
        c0, c1 = lay.col0[me], lay.col0[me + 1]
        z = fwd_recv.numpy().view(np.complex128).reshape(H, lay.pitch[me])[:, : c1 - c0]
        wx = 2.0 - 2.0 * np.cos(2.0 * np.pi * np.arange(c0, c1) / W)
        wy = 2.0 - 2.0 * np.cos(2.0 * np.pi * np.arange(H) / H)
        denom = 1.0 + self.c * self.lam / 2.0 * (wy[:, None] + wx[None, :])
        Y = np.fft.ifft(np.fft.fft(z, axis=0) / denom, axis=0) / W
        out = self._blocks(rev_send, lambda p: lay.row0[p + 1] - lay.row0[p] + 2, lambda p: lay.pitch[me], lay.P)
        for p in range(lay.P):
            rows = D.halo_rows(H, lay.row0[p], lay.row0[p + 1])
            out[p][:, : c1 - c0] = Y[rows]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, cases, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        for ci, (H, W, pen_kind) in enumerate(cases):
            pen = Charbonnier(0.8, 1e-4) if pen_kind == 0 else Welsch(0.2)
            params = SmoothParams(pen, 1.5, iters=4)
            cp = params.c_params()
            plan, lay = D.slab_layout(H, W, cp, _lib.ILS_F64, world, rank, device=-1)
            _lib.lib().ils_plan_destroy(plan)
            f = np.random.default_rng(7).random((H, W))
            f_ext = torch.from_numpy(np.ascontiguousarray(f[D.halo_rows(H, lay.row0[rank], lay.row0[rank + 1])]))
            kern = RefSlabKernels(lay, pen, params.lam, params.curvature)
            sm = D.SlabSmoother(lay, params.iters, kern, D.torch_exchange(),
                                lambda n: torch.zeros(n, dtype=torch.float64))
            u = torch.zeros((lay.rows, W), dtype=torch.float64)
            status = [_lib.STATUS_CLEAN]
            sm.smooth(f_ext, u, status)
            q.put((ci, rank, lay.row0[rank], u.numpy().copy(), status[0]))
    finally:
        dist.destroy_process_group()


def _worker_pipeline(rank, world, port, cases, q):
    """SlabPipeline: the planes of one image with overlapped (async) exchanges."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        for ci, (H, W, pen_kind) in enumerate(cases):
            pen = Charbonnier(0.8, 1e-4) if pen_kind == 0 else Welsch(0.2)
            params = SmoothParams(pen, 1.5, iters=3)
            plan, lay = D.slab_layout(H, W, params.c_params(), _lib.ILS_F64, world, rank, device=-1)
            _lib.lib().ils_plan_destroy(plan)
            rows = D.halo_rows(H, lay.row0[rank], lay.row0[rank + 1])
            planes = [np.random.default_rng(11 + c).random((H, W)) for c in range(3)]
            f_exts = [torch.from_numpy(np.ascontiguousarray(p[rows])) for p in planes]
            kern = RefSlabKernels(lay, pen, params.lam, params.curvature)
            pipe = D.SlabPipeline(lay, params.iters, kern, D.torch_exchange_async(),
                                  lambda n: torch.zeros(n, dtype=torch.float64), planes=3)
            us = [torch.zeros((lay.rows, W), dtype=torch.float64) for _ in range(3)]
            status = [_lib.STATUS_CLEAN]
            pipe.smooth(f_exts, us, status)
            q.put((ci, rank, lay.row0[rank], np.stack([u.numpy() for u in us]), status[0]))
    finally:
        dist.destroy_process_group()


def _run_world(world, cases, target=None):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=target or _worker, args=(r, world, port, cases, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = {}
    for _ in range(world * len(cases)):
        ci, rank, r0, u, status = q.get(timeout=240)
        got.setdefault(ci, []).append((r0, u, status))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return got


@pytest.mark.parametrize("world,cases", [(2, [(24, 20, 0), (9, 12, 1)]), (3, [(25, 18, 1)])])
def test_slab_driver_matches_single_image_oracle(world, cases):
    from oracle import ils_oracle as O

    got = _run_world(world, cases)
    for ci, (H, W, pen_kind) in enumerate(cases):
        parts = sorted(got[ci], key=lambda t: t[0])
        u = np.concatenate([p[1] for p in parts])
        assert all(p[2] == _lib.STATUS_CLEAN for p in parts)
        f = np.random.default_rng(7).random((H, W))
        spec = O.Charbonnier(0.8, 1e-4) if pen_kind == 0 else O.Welsch(0.2)
        ref = O.smooth_plane(f, spec, 1.5, 4)
        assert u.shape == ref.shape
        assert np.max(np.abs(u - ref)) < 1e-12, (H, W, world)


@pytest.mark.parametrize("world", [2, 3])
def test_slab_pipeline_overlapped_planes_match_oracle(world):
    from oracle import ils_oracle as O

    cases = [(18, 16, 0)]
    got = _run_world(world, cases, target=_worker_pipeline)
    H, W, _ = cases[0]
    parts = sorted(got[0], key=lambda t: t[0])
    u = np.concatenate([p[1] for p in parts], axis=1)  # [3, H, W]
    assert all(p[2] == _lib.STATUS_CLEAN for p in parts)
    for c in range(3):
        f = np.random.default_rng(11 + c).random((H, W))
        ref = O.smooth_plane(f, O.Charbonnier(0.8, 1e-4), 1.5, 3)
        assert np.max(np.abs(u[c] - ref)) < 1e-12, (world, c)


def test_frame_shard_partitions():
    for F, P in ((256, 8), (256, 3), (5, 8), (16, 1)):
        got = [list(D.frame_shard(F, P, r)) for r in range(P)]
        assert sum(got, []) == list(range(F))
        assert max(map(len, got)) - min(map(len, got)) <= 1


def test_slab_layout_counts_are_consistent():
    # rank r's fwd send to q equals q's fwd recv from r, for every pair (C planner)
    prm = SmoothParams(Welsch(10 / 255), 30.0, iters=10, c=2.0).c_params()
    for P in (2, 4, 8):
        lays = []
        for r in range(P):
            h, lay = D.slab_layout(4320, 7680, prm, _lib.ILS_F32, P, r, device=-1)
            _lib.lib().ils_plan_destroy(h)
            lays.append(lay)
        for r in range(P):
            for q in range(P):
                assert lays[r].counts[0][q] == lays[q].counts[1][r]
                assert lays[r].counts[2][q] == lays[q].counts[3][r]
        assert lays[0].row0[-1] == 4320 and lays[0].col0[-1] == 3841
        assert all(p % 2 == 0 for p in lays[0].pitch)
