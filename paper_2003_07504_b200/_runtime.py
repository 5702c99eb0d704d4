"""Device plumbing: plan cache, workspaces, host<->device moves (torch).

torch provides device memory, streams and the caching allocator; every
arithmetic step of the smoothing path is a kernel in libils_b200.so called
through the C ABI (_lib.py).  Nothing here computes on the CPU, and nothing
falls back: without CUDA the calls raise.
"""

from __future__ import annotations

import ctypes as C
import os
import threading
from collections import OrderedDict

import numpy as np

from . import _lib
from .errors import NumericalError

_PRECISION = os.environ.get("ILS_PRECISION", "fp32")
_plans: "OrderedDict[tuple, DevicePlan]" = OrderedDict()
_plans_lock = threading.Lock()
_MAX_PLANS = 32


def set_default_precision(p: str) -> None:
    """'fp32' (default, the throughput path) or 'fp64' (tight parity)."""
    global _PRECISION
    if p not in ("fp32", "fp64"):
        raise ValueError(f"precision must be 'fp32' or 'fp64', got {p!r}")
    _PRECISION = p


def get_default_precision() -> str:
    return _PRECISION


def _torch():
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("paper_2003_07504_b200 needs a CUDA device (sm_100a); there is no CPU fallback")
    return torch


def torch_dtype(precision):
    torch = _torch()
    precision = precision or _PRECISION
    if precision == "fp32":
        return torch.float32
    if precision == "fp64":
        return torch.float64
    raise ValueError(f"precision must be 'fp32' or 'fp64', got {precision!r}")


class DevicePlan:
    """Owns one ils_plan* (make_plan analogue, solver.py:78-106)."""

    def __init__(self, batch, height, width, cparams, dtype_code, device_index):
        L = _lib.lib()
        h = C.c_void_p()
        if isinstance(cparams, _lib.HqsParams):  # penalty-splitting baseline (hqs.py)
            _lib.check(L.ils_hqs_plan_create(C.byref(h), batch, height, width, C.byref(cparams), dtype_code,
                                             device_index), "ils_hqs_plan_create")
        else:
            _lib.check(L.ils_plan_create(C.byref(h), batch, height, width, C.byref(cparams), dtype_code,
                                         device_index), "ils_plan_create")
        self.ptr = h
        self.batch, self.height, self.width = batch, height, width
        self.dtype_code = dtype_code
        self.iters = cparams.iters
        ws = C.c_size_t()
        _lib.check(L.ils_workspace_size(h, C.byref(ws)), "ils_workspace_size")
        self.workspace_bytes = ws.value
        info = _lib.PlanInfo()
        _lib.check(L.ils_plan_get_info(h, C.byref(info)), "ils_plan_get_info")
        self.info = info.as_dict()

    def __del__(self):
        try:
            if getattr(self, "ptr", None):
                _lib.lib().ils_plan_destroy(self.ptr)
                self.ptr = None
        except Exception:
            pass


def get_plan(batch, height, width, cparams, dtype_code, device_index) -> DevicePlan:
    key = (batch, height, width, type(cparams).__name__) + tuple(getattr(cparams, n) for n, _ in cparams._fields_) + (
        dtype_code, device_index)
    with _plans_lock:
        plan = _plans.get(key)
        if plan is None:
            plan = DevicePlan(batch, height, width, cparams, dtype_code, device_index)
            _plans[key] = plan
            while len(_plans) > _MAX_PLANS:
                _plans.popitem(last=False)
        else:
            _plans.move_to_end(key)
        return plan


def plan_supported(height, width, precision) -> bool:
    """Whether the planner has a launch configuration for this plane size (host-only plan, no GPU work)."""
    L = _lib.lib()
    h = C.c_void_p()
    code = _lib.ILS_F32 if precision == "fp32" else _lib.ILS_F64
    st = L.ils_plan_create(C.byref(h), 1, height, width, C.byref(_dummy_params()), code, -1)
    if st == _lib.ILS_OK:
        L.ils_plan_destroy(h)
    return st == _lib.ILS_OK


def _stream_ptr(torch, device):
    return C.c_void_p(torch.cuda.current_stream(device).cuda_stream)


def smooth_device(f, cparams, trace=False, check=True):
    """All ILS iterations on a CUDA tensor f[B, H, W] (one launch sequence).

    Returns (u, energies[(iters+1), B] or None, status tensor).  With
    check=True the status word is read back and mapped to the reference's
    exceptions (ValueError for a non-finite input plane, NumericalError for
    a non-finite iterate, smoother.py:166-167).
    """
    torch = _torch()
    if f.dim() != 3 or not f.is_cuda:
        raise ValueError("smooth_device expects a CUDA tensor [B, H, W]")
    f = f.contiguous()
    B, H, W = f.shape
    code = _lib.ILS_F32 if f.dtype == torch.float32 else _lib.ILS_F64
    if f.dtype not in (torch.float32, torch.float64):
        raise ValueError(f"unsupported dtype {f.dtype}")
    f = _aligned(f)
    dev = f.device
    plan = get_plan(B, H, W, cparams, code, _dev_index(torch, dev))
    with torch.cuda.device(dev):
        u = torch.empty_like(f)
        ws = torch.empty(plan.workspace_bytes, dtype=torch.uint8, device=dev)
        status = torch.empty(1, dtype=torch.int32, device=dev)
        energies = torch.empty((cparams.iters + 1, B), dtype=torch.float64, device=dev) if trace else None
        L = _lib.lib()
        _lib.check(L.ils_smooth(plan.ptr, C.c_void_p(f.data_ptr()), C.c_void_p(u.data_ptr()), H * W,
                                C.c_void_p(ws.data_ptr()), _stream_ptr(torch, dev), C.c_void_p(status.data_ptr()),
                                C.c_void_p(energies.data_ptr()) if trace else None), "ils_smooth")
    if check:
        raise_status(int(status.item()))
    return u, energies, status


def _dev_index(torch, dev):
    return dev.index if dev.index is not None else torch.cuda.current_device()


def _aligned(t):
    """The row passes move whole rows with TMA bulk copies (16-byte aligned
    rows): a view at an odd storage offset is copied into fresh storage."""
    return t if t.data_ptr() % 16 == 0 else t.clone()


def raise_status(s: int) -> None:
    if s == _lib.STATUS_CLEAN:
        return
    if s == 0:
        raise ValueError("image plane contains non-finite values")
    raise NumericalError(f"non-finite iterate at iteration {s}")


def solve_device(f, mx, my, cparams):
    """solve_ls on CUDA tensors [B, H, W] (solver.py:109-134)."""
    torch = _torch()
    f, mx, my = (_aligned(t.contiguous()) for t in (f, mx, my))
    if not (f.shape == mx.shape == my.shape and f.dtype == mx.dtype == my.dtype and f.device == mx.device == my.device):
        raise ValueError("f, mu_x and mu_y must share shape, dtype and device")
    if f.dtype not in (torch.float32, torch.float64):
        raise ValueError(f"unsupported dtype {f.dtype}")
    B, H, W = f.shape
    code = _lib.ILS_F32 if f.dtype == torch.float32 else _lib.ILS_F64
    dev = f.device
    plan = get_plan(B, H, W, cparams, code, _dev_index(torch, dev))
    with torch.cuda.device(dev):
        u = torch.empty_like(f)
        ws = torch.empty(plan.workspace_bytes, dtype=torch.uint8, device=dev)
        status = torch.empty(1, dtype=torch.int32, device=dev)
        L = _lib.lib()
        _lib.check(L.ils_solve_ls(plan.ptr, C.c_void_p(f.data_ptr()), C.c_void_p(mx.data_ptr()),
                                  C.c_void_p(my.data_ptr()), C.c_void_p(u.data_ptr()), H * W,
                                  C.c_void_p(ws.data_ptr()), _stream_ptr(torch, dev), C.c_void_p(status.data_ptr())),
                   "ils_solve_ls")
    s = int(status.item())
    if s != _lib.STATUS_CLEAN:
        raise NumericalError(f"non-finite values in {('f', 'mu_x', 'mu_y')[s - 1]}")
    return u


def rfft2_device(x, cparams=None):
    """Hand-written real 2-D FFT of x[B, H, W] -> complex [B, H, W//2+1]."""
    torch = _torch()
    x = _aligned(x.contiguous())
    B, H, W = x.shape
    code = _lib.ILS_F32 if x.dtype == torch.float32 else _lib.ILS_F64
    cparams = cparams or _dummy_params()
    plan = get_plan(B, H, W, cparams, code, _dev_index(torch, x.device))
    pitch = plan.info["spec_pitch"]
    cdt = torch.complex64 if code == _lib.ILS_F32 else torch.complex128
    with torch.cuda.device(x.device):
        spec = torch.empty((B, H, pitch), dtype=cdt, device=x.device)
        _lib.check(_lib.lib().ils_rfft2(plan.ptr, C.c_void_p(x.data_ptr()), H * W, C.c_void_p(spec.data_ptr()),
                                        pitch, _stream_ptr(torch, x.device)), "ils_rfft2")
    return spec[:, :, : W // 2 + 1]


def irfft2_device(spec, width, cparams=None):
    """Inverse of rfft2_device (normalised like numpy.fft.irfft2)."""
    torch = _torch()
    B, H, Wc = spec.shape
    code = _lib.ILS_F32 if spec.dtype == torch.complex64 else _lib.ILS_F64
    cparams = cparams or _dummy_params()
    plan = get_plan(B, H, width, cparams, code, _dev_index(torch, spec.device))
    pitch = plan.info["spec_pitch"]
    with torch.cuda.device(spec.device):
        buf = torch.zeros((B, H, pitch), dtype=spec.dtype, device=spec.device)
        buf[:, :, :Wc] = spec
        rdt = torch.float32 if code == _lib.ILS_F32 else torch.float64
        x = torch.empty((B, H, width), dtype=rdt, device=spec.device)
        _lib.check(_lib.lib().ils_irfft2(plan.ptr, C.c_void_p(buf.data_ptr()), pitch, C.c_void_p(x.data_ptr()),
                                         H * width, _stream_ptr(torch, spec.device)), "ils_irfft2")
    return x


def _dummy_params():
    return _lib.Params(_lib.ILS_WELSCH, 0.0, 0.0, 1.0, 1.0, 2.0, 1)


def rgb_yuv_(planes, inverse: bool) -> None:
    """In-place BT.601 conversion of CUDA planes [F*3, H, W] (image.py:110-128)."""
    torch = _torch()
    n3, H, W = planes.shape
    code = _lib.ILS_F32 if planes.dtype == torch.float32 else _lib.ILS_F64
    _lib.check(_lib.lib().ils_rgb_yuv(C.c_void_p(planes.data_ptr()), code, H * W, H * W, n3 // 3, int(inverse),
                                      _stream_ptr(torch, planes.device)), "ils_rgb_yuv")


# Host staging for the numpy drop-in path: per-thread pinned buffers reused
# across calls (a fresh pageable stack + pageable copies cost ~4x the GPU
# work for a 1080p RGB image), the per-plane host copies / f32 -> f64
# widening spread over a few threads (numpy releases the GIL).
_tls = threading.local()
_pool = None
# host threads for staging copies (np.copyto releases the GIL)
_HOST_THREADS = int(os.environ.get("ILS_HOST_THREADS", "0")) or min(8, os.cpu_count() or 1)
# staging chunk: small enough that the first DMA starts early, large enough
# that per-copy launch cost stays negligible
_CHUNK_BYTES = int(float(os.environ.get("ILS_CHUNK_MB", "4")) * (1 << 20))
# fp32 targets: narrow f64 -> f32 in the staging copy (numpy's cast rounds to
# nearest-even exactly like the device's ils_convert, tests/test_gpu_host_staging.py)
# -- half the bytes over PCIe and half the pinned writes: 1080p RGB staging
# 2.0 -> 1.5 ms.  ILS_HOST_NARROW=0 stages f64 and narrows on the device.
_HOST_NARROW = os.environ.get("ILS_HOST_NARROW", "1") == "1"


_pool_lock = threading.Lock()


def _host_pool():
    global _pool
    with _pool_lock:
        if _pool is None:
            from concurrent.futures import ThreadPoolExecutor

            _pool = ThreadPoolExecutor(max_workers=_HOST_THREADS, thread_name_prefix="ils-host")
    return _pool


def _pinned(name, shape, dtype):
    """Per-thread pinned staging buffer `name`, reused across calls.

    A buffer handed out again first waits for the asynchronous copy that last
    read or wrote it (the event recorded by _pinned_done), so a host write
    into it can never race an in-flight DMA of the previous call.
    """
    torch = _torch()
    cache = getattr(_tls, "pinned", None)
    if cache is None:
        cache = _tls.pinned = {}
    buf, ev = cache.get(name, (None, None))
    if ev is not None:
        ev.synchronize()
    n = int(np.prod(shape))
    if buf is None or buf.numel() < n or buf.dtype != dtype:
        buf = torch.empty(max(n, 1), dtype=dtype, pin_memory=True)
    cache[name] = (buf, None)
    return buf[:n].view(*shape)


def _pinned_done(name, stream):
    """Record that `stream`'s queued copy is the last user of staging buffer `name`."""
    torch = _torch()
    buf, _ = _tls.pinned[name]
    ev = torch.cuda.Event()
    ev.record(stream)
    _tls.pinned[name] = (buf, ev)


def _parallel(fn, n):
    if n <= 1:
        for i in range(n):
            fn(i)
        return
    list(_host_pool().map(fn, range(n)))


def _row_chunks(B, H, W, itemsize):
    rows = max(1, _CHUNK_BYTES // max(1, W * itemsize))
    return [(i, r0, min(H, r0 + rows)) for i in range(B) for r0 in range(0, H, rows)]


def to_device_planes(planes, precision=None):
    """Host planes -> one CUDA tensor [B, H, W] of the target dtype.

    The planes are staged in ~4 MB row chunks spread over the host pool: each
    worker copies its chunk into pinned memory and queues that chunk's
    host-to-device copy on the caller's stream at once, so the PCIe transfer
    of one chunk overlaps the host copies of the others.  fp32 targets are
    narrowed in the staging copy (_HOST_NARROW), or staged as f64 and
    narrowed on the device by the library's own kernel (ils_convert)."""
    torch = _torch()
    dt = torch_dtype(precision)
    arrs = [np.asarray(p, dtype=np.float64) for p in planes]
    B = len(arrs)
    H, W = arrs[0].shape
    stream = torch.cuda.current_stream()
    if dt == torch.float32 and _HOST_NARROW:
        dev = torch.empty((B, H, W), dtype=dt, device=stream.device)
        stage = _pinned("in32", (B, H, W), dt)
        host = stage.numpy()
        chunks = _row_chunks(B, H, W, 4)

        def one32(k):
            i, r0, r1 = chunks[k]
            np.copyto(host[i, r0:r1], arrs[i][r0:r1], casting="same_kind")
            with torch.cuda.stream(stream):
                dev[i, r0:r1].copy_(stage[i, r0:r1], non_blocking=True)

        _parallel(one32, len(chunks))
        _pinned_done("in32", stream)
        return dev
    dev = torch.empty((B, H, W), dtype=torch.float64, device=stream.device)
    stage = _pinned("in", (B, H, W), torch.float64)
    host = stage.numpy()
    chunks = _row_chunks(B, H, W, 8)

    def one(k):
        i, r0, r1 = chunks[k]
        np.copyto(host[i, r0:r1], arrs[i][r0:r1])
        with torch.cuda.stream(stream):
            dev[i, r0:r1].copy_(stage[i, r0:r1], non_blocking=True)

    _parallel(one, len(chunks))
    _pinned_done("in", stream)
    if dt == torch.float64:
        return dev
    out = torch.empty((B, H, W), dtype=dt, device=dev.device)  # narrowed by the library's own kernel
    _lib.check(_lib.lib().ils_convert(C.c_void_p(dev.data_ptr()), _lib.ILS_F64, C.c_void_p(out.data_ptr()),
                                      _lib.ILS_F32, dev.numel(), _stream_ptr(torch, dev.device)), "ils_convert")
    return out


# ---- result planes in pooled pinned memory
# The float64 planes a call returns are numpy views of a pinned buffer: the
# device widens u to f64 (ils_convert) and one DMA writes it straight into
# the caller's arrays -- no host-side widening pass and no page faults on
# fresh memory (1080p RGB result: 0.94 ms vs 2.6 ms for D2H of fp32 plus a
# threaded widening copy into new arrays).  The buffer returns to the pool
# when the last view of it dies.  Pinned bytes held by results are capped
# (ILS_PINNED_OUT_MB, default 1024); past the cap results are ordinary
# numpy arrays filled on the host.
_OUT_LIMIT = int(os.environ.get("ILS_PINNED_OUT_MB", "1024")) << 20


class _OutPool:
    def __init__(self):
        self.lock = threading.Lock()
        self.free = []  # pinned float64 tensors no result refers to
        self.total = 0  # bytes of every pooled buffer, free or leased

    def take(self, n):
        """A pinned float64 tensor of >= n elements, or None past the cap."""
        torch = _torch()
        with self.lock:
            best = None
            for k, t in enumerate(self.free):
                if t.numel() >= n and (best is None or t.numel() < self.free[best].numel()):
                    best = k
            if best is not None:
                return self.free.pop(best)
            while self.free and self.total + 8 * n > _OUT_LIMIT:
                self.total -= 8 * self.free.pop().numel()
            if self.total + 8 * n > _OUT_LIMIT:
                return None
            self.total += 8 * n
        return torch.empty(n, dtype=torch.float64, pin_memory=True)

    def give(self, t):
        with self.lock:
            self.free.append(t)


_out_pool = _OutPool()


class _Lease:
    """numpy base object of pooled result planes: returns the buffer on death."""

    __slots__ = ("_t", "__array_interface__")

    def __init__(self, t, shape):
        self._t = t
        self.__array_interface__ = {"shape": tuple(shape), "typestr": "<f8", "data": (t.data_ptr(), False),
                                    "version": 3}

    def __del__(self):
        try:
            _out_pool.give(self._t)
        except Exception:  # interpreter teardown
            pass


def to_host_f64(t):
    """CUDA planes [B, H, W] -> list of C-contiguous float64 numpy planes."""
    torch = _torch()
    t = t.detach()
    B, H, W = t.shape
    stream = torch.cuda.current_stream(t.device)
    buf = _out_pool.take(B * H * W) if t.is_contiguous() else None
    if buf is not None:
        try:
            if t.dtype == torch.float64:
                w = t
            else:
                w = torch.empty((B, H, W), dtype=torch.float64, device=t.device)
                _lib.check(_lib.lib().ils_convert(C.c_void_p(t.data_ptr()), _lib.ILS_F32, C.c_void_p(w.data_ptr()),
                                                  _lib.ILS_F64, t.numel(), _stream_ptr(torch, t.device)),
                           "ils_convert")
            buf[:B * H * W].view(B, H, W).copy_(w, non_blocking=True)
            stream.synchronize()  # the caller reads the arrays next: nothing left in flight
        except BaseException:
            _out_pool.give(buf)
            raise
        arr = np.asarray(_Lease(buf, (B, H, W)))
        return [arr[i] for i in range(B)]
    # past the cap: fresh arrays, widened on the host in row chunks
    stage = _pinned("out", (B, H, W), t.dtype)
    stage.copy_(t, non_blocking=True)
    stream.synchronize()
    host = stage.numpy()
    out = [np.empty((H, W), dtype=np.float64) for _ in range(B)]
    chunks = _row_chunks(B, H, W, 8)

    def one(k):
        i, r0, r1 = chunks[k]
        np.copyto(out[i][r0:r1], host[i, r0:r1])

    _parallel(one, len(chunks))
    return out


def _side_streams(dev):
    """Per-thread (staging, result) streams of device `dev` for smooth_planes_host."""
    torch = _torch()
    cache = getattr(_tls, "side", None)
    if cache is None:
        cache = _tls.side = {}
    key = _dev_index(torch, dev)
    if key not in cache:
        cache[key] = (torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev))
    return cache[key]


def smooth_planes_host(planes, cparams, precision=None):
    """Host float64 planes -> smoothed float64 planes, pipelined plane by plane.

    The reference's smooth_color smooths its channels independently
    (smoother.py:204-213), so each plane can start as soon as its own rows
    are staged: the chunk copies of all planes run on the host pool and
    their H2Ds on a staging stream; plane i's smooth (one launch sequence on
    the caller's stream) waits only for plane i's chunks, and its result
    widens on the device and goes to pooled pinned memory on a third stream
    while the next plane computes.  The arithmetic is exactly the batched
    path's (a plane's bits do not depend on its batch).  Returns None when
    the pinned result pool is over its cap (the caller uses the batched path).
    """
    torch = _torch()
    dt = torch_dtype(precision)
    arrs = [np.asarray(p, dtype=np.float64) for p in planes]
    B = len(arrs)
    H, W = arrs[0].shape
    n = B * H * W
    buf = _out_pool.take(n)
    if buf is None:
        return None
    cur = torch.cuda.current_stream()
    dev = cur.device
    s_in, s_out = _side_streams(dev)
    s_in.wait_stream(cur)
    narrow = dt == torch.float32 and _HOST_NARROW
    sdt = dt if narrow else torch.float64
    stage = _pinned("pipe_in", (B, H, W), sdt)
    host = stage.numpy()
    dev_in = torch.empty((B, H, W), dtype=sdt, device=dev)
    chunks = _row_chunks(B, H, W, 4 if narrow else 8)

    def one(k):
        i, r0, r1 = chunks[k]
        np.copyto(host[i, r0:r1], arrs[i][r0:r1], casting="same_kind")
        with torch.cuda.stream(s_in):
            dev_in[i, r0:r1].copy_(stage[i, r0:r1], non_blocking=True)

    pool = _host_pool()
    futs = [pool.submit(one, k) for k in range(len(chunks))]
    out = buf[:n].view(B, H, W)
    L = _lib.lib()
    keep, statuses = [], []
    ok = False
    try:
        for i in range(B):
            for f, (pi, _, _) in zip(futs, chunks):
                if pi == i:
                    f.result()
            ev = torch.cuda.Event()
            ev.record(s_in)  # after every H2D of plane i (queued by now)
            cur.wait_event(ev)
            fi = dev_in[i:i + 1]
            if sdt != dt:  # staged as f64: narrowed by the library's own kernel
                f32 = torch.empty((1, H, W), dtype=dt, device=dev)
                _lib.check(L.ils_convert(C.c_void_p(fi.data_ptr()), _lib.ILS_F64, C.c_void_p(f32.data_ptr()),
                                         _lib.ILS_F32, H * W, _stream_ptr(torch, dev)), "ils_convert")
                fi = f32
            u, _, st = smooth_device(fi, cparams, check=False)
            statuses.append(st)
            if u.dtype == torch.float64:
                w = u
            else:
                w = torch.empty((1, H, W), dtype=torch.float64, device=dev)
                _lib.check(L.ils_convert(C.c_void_p(u.data_ptr()), _lib.ILS_F32, C.c_void_p(w.data_ptr()),
                                         _lib.ILS_F64, H * W, _stream_ptr(torch, dev)), "ils_convert")
            done = torch.cuda.Event()
            done.record(cur)
            s_out.wait_event(done)
            with torch.cuda.stream(s_out):
                out[i:i + 1].copy_(w, non_blocking=True)
            keep.append((fi, u, w))  # alive until the result stream is drained
        ok = True
    finally:
        for f in futs:
            f.exception()  # wait for every staging task (a failed one re-raises in the loop)
        s_out.synchronize()
        cur.synchronize()
        _pinned_done("pipe_in", s_in)
        if not ok:
            _out_pool.give(buf)  # nothing in flight into it, and no result refers to it
    arr = np.asarray(_Lease(buf, (B, H, W)))
    for st in statuses:  # in plane order, as the batched path reports them
        raise_status(int(st.item()))
    return [arr[i] for i in range(B)]


def smooth_device_u8(frames, cparams, precision=None, check=True):
    """8-bit interleaved frames uint8[F, H, W, C] on the GPU -> same layout (ils_smooth_u8).

    Equals quantising (floor(clip01(u) 255 + 0.5), formats.py:25-27) the
    smoothing of the planes v / 255 (formats.py read side); the conversions
    run inside the first and last row passes.
    """
    torch = _torch()
    if frames.dim() != 4 or not frames.is_cuda or frames.dtype != torch.uint8:
        raise ValueError("smooth_device_u8 expects a CUDA uint8 tensor [F, H, W, C]")
    frames = frames.contiguous()
    F, H, W, Ch = frames.shape
    code = _lib.ILS_F32 if (precision or _PRECISION) == "fp32" else _lib.ILS_F64
    dev = frames.device
    plan = get_plan(F * Ch, H, W, cparams, code, _dev_index(torch, dev))
    with torch.cuda.device(dev):
        u = torch.empty_like(frames)
        ws = torch.empty(plan.workspace_bytes, dtype=torch.uint8, device=dev)
        status = torch.empty(1, dtype=torch.int32, device=dev)
        _lib.check(_lib.lib().ils_smooth_u8(plan.ptr, C.c_void_p(frames.data_ptr()), C.c_void_p(u.data_ptr()), Ch,
                                            C.c_void_p(ws.data_ptr()), _stream_ptr(torch, dev),
                                            C.c_void_p(status.data_ptr())), "ils_smooth_u8")
    if check:
        raise_status(int(status.item()))
    return u


# Standalone field kernels (grad_x / grad_y / adjoint_accumulate / aux_update /
# energy of the reference API): numpy in -> float64 on the device -> fresh
# float64 numpy out; CUDA tensors in -> tensors of the same dtype out.
def _as_field(a):
    """(CUDA tensor [B, H, W] or [n], was_numpy, original shape)."""
    torch = _torch()
    if isinstance(a, torch.Tensor):
        if not a.is_cuda:
            a = a.to("cuda")
        if a.dtype not in (torch.float32, torch.float64):
            a = a.to(torch.float64)
        return a.contiguous(), False, tuple(a.shape)
    arr = np.asarray(a, dtype=np.float64)
    return torch.from_numpy(np.ascontiguousarray(arr)).to("cuda"), True, arr.shape


def _planes3(t):
    if t.dim() == 2:
        return t.unsqueeze(0)
    if t.dim() == 3:
        return t
    raise ValueError(f"expected a 2-D plane or a [B, H, W] stack, got shape {tuple(t.shape)}")


def _dtype_code(t):
    torch = _torch()
    return _lib.ILS_F32 if t.dtype == torch.float32 else _lib.ILS_F64


def _out(t, was_np, shape):
    return t.cpu().numpy().reshape(shape) if was_np else t.reshape(shape)


def grad_fields(u, which):
    """which: 'x' or 'y' (solver.py:33-40)."""
    torch = _torch()
    t, was_np, shape = _as_field(u)
    p = _planes3(t)
    B, H, W = p.shape
    out = torch.empty_like(p)
    gx, gy = (out, None) if which == "x" else (None, out)
    with torch.cuda.device(p.device):
        _lib.check(_lib.lib().ils_grad(C.c_void_p(p.data_ptr()), C.c_void_p(gx.data_ptr()) if gx is not None else None,
                                       C.c_void_p(gy.data_ptr()) if gy is not None else None, B, H, W, H * W,
                                       _dtype_code(p), _stream_ptr(torch, p.device)), "ils_grad")
    return _out(out, was_np, shape)


def adjoint_fields(mu_x, mu_y):
    """solver.py:43-49."""
    torch = _torch()
    tx, was_np, shape = _as_field(mu_x)
    ty, _, shape_y = _as_field(mu_y)
    if shape != shape_y:
        raise ValueError(f"field shapes differ: {shape} vs {shape_y}")
    if ty.dtype != tx.dtype:
        ty = ty.to(tx.dtype)
    px, py = _planes3(tx), _planes3(ty.to(tx.device))
    B, H, W = px.shape
    out = torch.empty_like(px)
    with torch.cuda.device(px.device):
        _lib.check(_lib.lib().ils_adjoint_accumulate(C.c_void_p(px.data_ptr()), C.c_void_p(py.data_ptr()),
                                                     C.c_void_p(out.data_ptr()), B, H, W, H * W, _dtype_code(px),
                                                     _stream_ptr(torch, px.device)), "ils_adjoint_accumulate")
    return _out(out, was_np, shape)


def aux_fields(cparams, x):
    """penalty.py:117-126 on every element of x."""
    torch = _torch()
    t, was_np, shape = _as_field(x)
    out = torch.empty_like(t)
    with torch.cuda.device(t.device):
        _lib.check(_lib.lib().ils_aux_update(C.byref(cparams), C.c_void_p(t.data_ptr()), C.c_void_p(out.data_ptr()),
                                             t.numel(), _dtype_code(t), _stream_ptr(torch, t.device)),
                   "ils_aux_update")
    return _out(out, was_np, shape)


def energy_fields(cparams, u, f):
    """smoother.py:93-101: one float (2-D input) or a float64 tensor [B] (stacked tensors)."""
    torch = _torch()
    tu, was_np, shape = _as_field(u)
    tf, _, shape_f = _as_field(f)
    if shape != shape_f:
        raise ValueError(f"shapes differ: u {shape}, f {shape_f}")
    if tf.dtype != tu.dtype:
        tf = tf.to(tu.dtype)
    pu, pf = _planes3(tu), _planes3(tf.to(tu.device))
    B, H, W = pu.shape
    out = torch.empty(B, dtype=torch.float64, device=pu.device)
    scratch = torch.empty(B * 256 * 3, dtype=torch.float64, device=pu.device)
    with torch.cuda.device(pu.device):
        _lib.check(_lib.lib().ils_energy(C.byref(cparams), C.c_void_p(pu.data_ptr()), C.c_void_p(pf.data_ptr()), B, H,
                                         W, H * W, _dtype_code(pu), C.c_void_p(out.data_ptr()),
                                         C.c_void_p(scratch.data_ptr()), _stream_ptr(torch, pu.device)), "ils_energy")
    if len(shape) == 2:
        return float(out[0].item())
    return out


def denominator(height, width, lam, c):
    """SolverPlan.denom (solver.py:100-102) as a float64 numpy array, evaluated on the GPU."""
    torch = _torch()
    out = torch.empty((height, width), dtype=torch.float64, device="cuda")
    _lib.check(_lib.lib().ils_denominator(C.c_void_p(out.data_ptr()), height, width, float(lam), float(c),
                                          _stream_ptr(torch, out.device)), "ils_denominator")
    return out.cpu().numpy()


def fft2_full(f):
    """fft2 of a real plane as the reference caches it (SolverPlan.with_data,
    solver.py:69-75): complex128 H x W, from the hand-written fp64 r2c on the
    GPU, the other half filled in by Hermitian symmetry X[k1, k2] =
    conj(X[-k1 mod H, W - k2])."""
    torch = _torch()
    x = torch.from_numpy(np.ascontiguousarray(np.asarray(f, dtype=np.float64))).to("cuda")
    H, W = x.shape
    try:
        half = rfft2_device(x[None])[0]  # [H, W//2 + 1] view of rows spec_pitch apart
        pitch = half.stride(0)
    except ValueError:
        # no fp64 plan for this size (fp64 lines stop at about 4096 points):
        # the fp32 transform, widened (relative error ~1e-7)
        h32 = rfft2_device(x[None].float())[0]
        pitch = h32.stride(0)
        half = torch.empty((H, pitch), dtype=torch.complex128, device=x.device)
        _lib.check(_lib.lib().ils_convert(C.c_void_p(h32.data_ptr()), _lib.ILS_F32, C.c_void_p(half.data_ptr()),
                                          _lib.ILS_F64, 2 * H * pitch, _stream_ptr(torch, x.device)), "ils_convert")
    full = torch.empty((H, W), dtype=torch.complex128, device=x.device)
    _lib.check(_lib.lib().ils_hermitian_full(C.c_void_p(half.data_ptr()), pitch, C.c_void_p(full.data_ptr()), H, W,
                                             _stream_ptr(torch, x.device)), "ils_hermitian_full")
    return full.cpu().numpy()
