"""The pipelined HOST-buffer entry points of the C ABI, frame by frame (needs a B200).

ils_smooth_host / ils_smooth_host_u8 (csrc/ils_api.cu host_pipeline) run
consecutive batches on two compute lanes through four I/O slots, each slot's
batch replayed from a CUDA graph cached per (thread, plan, buffers).  These
tests cover every lane and slot (nbatches >= 6), graph-cache reuse across
calls and across plans on one thread, and the status decoding: every frame
must be bit-identical to the device-resident ils_smooth / smooth_frames_u8
result of the same frame (the reference contract is smooth_color per image,
pkg/src/ilsmooth/smoother.py:175-217; 8-bit I/O formats.py:25-27).
"""

import ctypes as C

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs CUDA")]

import paper_2003_07504_b200 as ils  # noqa: E402
from paper_2003_07504_b200 import _lib, _runtime as rt  # noqa: E402

PARAMS = ils.SmoothParams(ils.Charbonnier(0.8, 1e-4), 1.0, iters=4)


class HostRunner:
    """One plan + its workspace and host-I/O device buffer, called through the C ABI."""

    def __init__(self, batch, H, W, params=PARAMS):
        self.plan = rt.get_plan(batch, H, W, params.c_params(), _lib.ILS_F32, 0)
        L = _lib.lib()
        io = C.c_size_t()
        _lib.check(L.ils_host_io_size(self.plan.ptr, C.byref(io)), "ils_host_io_size")
        self.ws = torch.empty(self.plan.workspace_bytes, dtype=torch.uint8, device="cuda")
        self.io = torch.empty(io.value, dtype=torch.uint8, device="cuda")
        self.B, self.H, self.W = batch, H, W

    def run_f32(self, fh, uh, nb):
        bad = C.c_int32(-7)
        rc = _lib.lib().ils_smooth_host(self.plan.ptr, C.c_void_p(fh.data_ptr()), C.c_void_p(uh.data_ptr()),
                                        self.H * self.W, nb, C.c_void_p(self.ws.data_ptr()),
                                        C.c_void_p(self.io.data_ptr()),
                                        C.c_void_p(torch.cuda.current_stream().cuda_stream), C.byref(bad))
        return rc, bad.value

    def run_u8(self, fh, uh, ch, nb):
        bad = C.c_int32(-7)
        rc = _lib.lib().ils_smooth_host_u8(self.plan.ptr, C.c_void_p(fh.data_ptr()), C.c_void_p(uh.data_ptr()), ch,
                                           nb, C.c_void_p(self.ws.data_ptr()), C.c_void_p(self.io.data_ptr()),
                                           C.c_void_p(torch.cuda.current_stream().cuda_stream), C.byref(bad))
        return rc, bad.value


def _pinned_rand(shape, seed, dtype=torch.float32):
    g = torch.Generator().manual_seed(seed)
    t = torch.empty(shape, dtype=dtype, pin_memory=True)
    if dtype == torch.uint8:
        t.copy_(torch.randint(0, 256, shape, generator=g, dtype=torch.uint8))
    else:
        t.copy_(torch.rand(shape, generator=g, dtype=dtype))
    return t


def _device_ref(fh_batches):
    """Each batch smoothed alone by ils_smooth on the device (smooth_batch)."""
    return torch.stack([ils.smooth_batch(b.to("cuda"), PARAMS).cpu() for b in fh_batches])


@pytest.mark.parametrize("nb", [7, 9])
def test_host_f32_every_frame_every_lane_and_slot(nb):
    CH, H, W = 3, 270, 480
    R = HostRunner(CH, H, W)
    for call, seed in enumerate((11, 12)):  # second call replays the cached slot graphs on new data
        fh = _pinned_rand((nb, CH, H, W), seed)
        uh = torch.full((nb, CH, H, W), float("nan"), pin_memory=True)
        rc, bad = R.run_f32(fh, uh, nb)
        assert rc == _lib.ILS_OK and bad == -1, (call, rc, _lib.last_error())
        ref = _device_ref(list(fh))
        for k in range(nb):  # batch k ran on lane k & 1 through I/O slot k % 4
            assert torch.equal(uh[k], ref[k]), (call, k)


def test_host_f32_second_plan_on_same_thread_then_back():
    CH = 3
    A = HostRunner(CH, 270, 480)
    Bp = HostRunner(CH, 135, 240)
    for R, seed in ((A, 1), (Bp, 2), (A, 3), (Bp, 4)):
        nb = 6
        fh = _pinned_rand((nb, CH, R.H, R.W), seed)
        uh = torch.empty((nb, CH, R.H, R.W), pin_memory=True)
        rc, bad = R.run_f32(fh, uh, nb)
        assert rc == _lib.ILS_OK and bad == -1
        ref = _device_ref(list(fh))
        assert torch.equal(uh, ref), (R.H, seed)


def test_host_f32_nonfinite_frame_in_batch_5():
    CH, H, W, nb = 3, 96, 128, 7
    R = HostRunner(CH, H, W)
    fh = _pinned_rand((nb, CH, H, W), 5)
    fh[5, 1, 10, 17] = float("nan")
    uh = torch.empty_like(fh).pin_memory()
    rc, bad = R.run_f32(fh, uh, nb)
    assert rc == _lib.ILS_ENONFINITE_INPUT and bad == 0
    with pytest.raises(ValueError, match="non-finite"):
        _lib.check(rc, "ils_smooth_host")
    # the clean batches around it still hold their results
    ref = _device_ref([fh[k] for k in (4, 6)])
    assert torch.equal(uh[4], ref[0]) and torch.equal(uh[6], ref[1])
    # and the pipeline is reusable after the error
    fh[5, 1, 10, 17] = 0.5
    rc, bad = R.run_f32(fh, uh, nb)
    assert rc == _lib.ILS_OK and bad == -1


@pytest.mark.parametrize("frames_per_batch", [1, 2])
def test_host_u8_every_frame_matches_device_path(frames_per_batch):
    CH, H, W, nb = 3, 270, 480, 7
    R = HostRunner(CH * frames_per_batch, H, W)
    for seed in (21, 22):
        fh = _pinned_rand((nb * frames_per_batch, H, W, CH), seed, torch.uint8)
        uh = torch.zeros_like(fh).pin_memory()
        rc, bad = R.run_u8(fh, uh, CH, nb)
        assert rc == _lib.ILS_OK and bad == -1, _lib.last_error()
        for k in range(nb * frames_per_batch):
            ref = ils.smooth_frames_u8(fh[k].to("cuda"), PARAMS).cpu()
            assert torch.equal(uh[k], ref), (seed, k)


def test_host_u8_1080p_two_lanes_all_slots():
    # the bench's e2e configuration (1080p RGB, 1 frame per batch), 6 batches
    CH, H, W, nb = 3, 1080, 1920, 6
    R = HostRunner(CH, H, W)
    fh = _pinned_rand((nb, H, W, CH), 31, torch.uint8)
    uh = torch.zeros_like(fh).pin_memory()
    rc, bad = R.run_u8(fh, uh, CH, nb)
    assert rc == _lib.ILS_OK and bad == -1
    ref = ils.smooth_frames_u8(fh.to("cuda"), PARAMS).cpu()
    for k in range(nb):
        assert torch.equal(uh[k], ref[k]), k
