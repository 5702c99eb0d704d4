"""Host staging of the numpy drop-in (needs a B200).

smooth_plane / smooth_color on float64 numpy planes (the reference's entry
points, smoother.py:132-217) stage the planes in row chunks over a host
thread pool and hand back float64 planes that are views of pooled pinned
buffers (_runtime.to_device_planes / to_host_f64).  The values must be
exactly what the device path computes on the same planes, for every chunk
geometry and input layout; live results never share a buffer; a dead
result's buffer is reused; past the pinned cap results are plain arrays.
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs CUDA")]

import paper_2003_07504_b200 as ils  # noqa: E402
from paper_2003_07504_b200 import _runtime as rt  # noqa: E402

PARAMS = ils.SmoothParams(ils.Charbonnier(0.8, 1e-4), 1.0, iters=3)


def _device_result(planes):
    f = torch.from_numpy(np.stack(planes)).to("cuda").float()
    u = ils.smooth_batch(f, PARAMS)
    return u.double().cpu().numpy()


@pytest.mark.parametrize("H,W,chunk", [(1080, 1920, None), (203, 1920, 3 * 1920 * 8), (77, 96, 1)])
def test_smooth_color_equals_device_path_for_every_chunking(H, W, chunk, monkeypatch):
    if chunk is not None:
        monkeypatch.setattr(rt, "_CHUNK_BYTES", chunk)
    rng = np.random.default_rng(H * W)
    planes = [rng.random((H, W)) for _ in range(3)]
    out = ils.smooth_color(ils.MultiImage(tuple(planes), ils.RGB), PARAMS)
    ref = _device_result(planes)
    for c in range(3):
        a = out.channels[c]
        assert a.dtype == np.float64 and a.shape == (H, W) and a.flags.c_contiguous
        assert not a.flags.writeable  # MultiImage freezes its channels (image.py:77)
        assert np.array_equal(a, ref[c])


def test_strided_and_foreign_dtype_inputs():
    rng = np.random.default_rng(3)
    big = rng.random((2 * 150, 2 * 256))
    view = big[::2, 1::2]  # non-contiguous plane
    a = ils.smooth_plane(view, PARAMS)
    b = ils.smooth_plane(np.ascontiguousarray(view), PARAMS)
    assert np.array_equal(a, b)
    c = ils.smooth_plane(view.astype(np.float32), PARAMS)  # widened by as_plane like the reference
    d = ils.smooth_plane(view.astype(np.float32).astype(np.float64), PARAMS)
    assert np.array_equal(c, d)


def _addr(a):
    return a.__array_interface__["data"][0]


def test_live_results_never_share_and_dead_ones_are_reused():
    rng = np.random.default_rng(5)
    f = rng.random((120, 640))
    r1 = ils.smooth_plane(f, PARAMS)
    keep = r1.copy()
    r2 = ils.smooth_plane(1.0 - f, PARAMS)
    assert not np.shares_memory(r1, r2)
    assert np.array_equal(r1, keep)  # the second call did not write into the live first result
    r1[:] = -1.0  # results are the caller's to modify
    r3 = ils.smooth_plane(f, PARAMS)
    assert np.array_equal(r3, keep) and not np.shares_memory(r1, r3)
    addr2 = _addr(r2)
    del r2
    r4 = ils.smooth_plane(f, PARAMS)
    assert _addr(r4) == addr2 and np.array_equal(r4, keep)
    # a larger result after smaller ones, then a smaller one again
    big = ils.smooth_plane(rng.random((300, 640)), PARAMS)
    del big
    r5 = ils.smooth_plane(f, PARAMS)
    assert np.array_equal(r5, keep)


def test_pinned_cap_falls_back_to_plain_arrays(monkeypatch):
    rng = np.random.default_rng(6)
    planes = [rng.random((64, 384)) for _ in range(3)]
    img = ils.MultiImage(tuple(planes), ils.RGB)
    pooled = ils.smooth_color(img, PARAMS)
    assert not pooled.channels[0].flags.owndata
    monkeypatch.setattr(rt, "_OUT_LIMIT", 0)
    monkeypatch.setattr(rt, "_out_pool", rt._OutPool())
    plain = ils.smooth_color(img, PARAMS)
    for c in range(3):
        assert plain.channels[c].flags.owndata and plain.channels[c].flags.c_contiguous
        assert np.array_equal(plain.channels[c], pooled.channels[c])


def test_luminance_and_fp64_paths_through_the_staging():
    rng = np.random.default_rng(7)
    planes = [rng.random((96, 200)) for _ in range(3)]
    img = ils.MultiImage(tuple(planes), ils.RGB)
    lum = ils.SmoothParams(ils.Charbonnier(0.8, 1e-4), 1.0, iters=3, color_mode=ils.ColorMode.LUMINANCE_ONLY)
    out = ils.smooth_color(img, lum)
    y = ils.rgb_to_yuv(img)
    ys = ils.smooth_plane(y.channels[0], lum)
    back = ils.yuv_to_rgb(ils.MultiImage((ys, y.channels[1], y.channels[2]), ils.YUV))
    for c in range(3):
        assert np.max(np.abs(out.channels[c] - back.channels[c])) < 1e-5
    a64 = ils.smooth_color(img, PARAMS, precision="fp64")
    f = torch.from_numpy(np.stack(planes)).to("cuda")
    ref = ils.smooth_batch(f, PARAMS).cpu().numpy()
    for c in range(3):
        assert np.array_equal(a64.channels[c], ref[c])


def test_host_narrowing_variant_is_bitwise_the_device_cast(monkeypatch):
    rng = np.random.default_rng(8)
    planes = [rng.random((130, 1920)) * 3 - 1 for _ in range(3)]
    img = ils.MultiImage(tuple(planes), ils.RGB)
    monkeypatch.setattr(rt, "_HOST_NARROW", False)  # f64 staged, narrowed by ils_convert
    a = ils.smooth_color(img, PARAMS)
    monkeypatch.setattr(rt, "_HOST_NARROW", True)
    monkeypatch.setattr(rt, "_CHUNK_BYTES", 7 * 1920 * 4)
    b = ils.smooth_color(img, PARAMS)
    for c in range(3):
        assert np.array_equal(a.channels[c], b.channels[c])


def test_pipelined_planes_equal_the_batched_path(monkeypatch):
    # smooth_color's per-channel pipeline (one launch sequence per plane,
    # staged and returned plane by plane) gives the batched path's bits
    rng = np.random.default_rng(9)
    planes = [rng.random((270, 480)) for _ in range(3)]
    img = ils.MultiImage(tuple(planes), ils.RGB)
    piped = ils.smooth_color(img, PARAMS)
    monkeypatch.setattr(rt, "smooth_planes_host", lambda *a, **k: None)  # force the batched path
    batched = ils.smooth_color(img, PARAMS)
    for c in range(3):
        assert np.array_equal(piped.channels[c], batched.channels[c])
    monkeypatch.undo()
    monkeypatch.setattr(rt, "_HOST_NARROW", False)
    piped64 = ils.smooth_color(img, PARAMS)  # staged as f64, narrowed on the device
    for c in range(3):
        assert np.array_equal(piped64.channels[c], batched.channels[c])
    fp64 = ils.smooth_color(img, PARAMS, precision="fp64")
    ref = ils.smooth_batch(torch.from_numpy(np.stack(planes)).to("cuda"), PARAMS).cpu().numpy()
    for c in range(3):
        assert np.array_equal(fp64.channels[c], ref[c])


def test_pipelined_planes_report_errors_in_channel_order():
    rng = np.random.default_rng(10)
    huge = ils.SmoothParams(ils.Charbonnier(0.8, 1e-4), 1e30, iters=3)
    planes = [rng.random((64, 96)) * 1e30 for _ in range(3)]
    img = ils.MultiImage(tuple(planes), ils.RGB)
    ils.smooth_color(img, PARAMS)  # a pooled buffer of this size exists
    before = rt._out_pool.total
    for _ in range(3):
        with pytest.raises(ils.NumericalError):
            ils.smooth_color(img, huge)
    ok = ils.smooth_color(img, PARAMS)
    assert ok.channels[0].shape == (64, 96)
    assert rt._out_pool.total == before  # failed calls returned their result buffers


def test_concurrent_callers_get_their_own_results():
    # per-thread staging buffers and streams, a shared host pool and result pool
    from concurrent.futures import ThreadPoolExecutor

    rng = np.random.default_rng(11)
    imgs = [ils.MultiImage(tuple(rng.random((150, 256)) for _ in range(3)), ils.RGB) for _ in range(8)]
    serial = [ils.smooth_color(im, PARAMS) for im in imgs]
    with ThreadPoolExecutor(4) as ex:
        for _ in range(2):
            par = list(ex.map(lambda im: ils.smooth_color(im, PARAMS), imgs))
            for a, b in zip(par, serial):
                for c in range(3):
                    assert np.array_equal(a.channels[c], b.channels[c])
