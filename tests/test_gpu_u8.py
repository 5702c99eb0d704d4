"""8-bit ingest/egress fused into the first/last row passes.

The reference's 8-bit path is read (v/255, formats.py:43) -> smooth_color ->
quantize (floor(clip01(u)*255+0.5), formats.py:25-27).  Goldens come from the
reference's own codec round trip (tests/golden/make_golden.py).
"""

import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2003_07504_b200 as ils  # noqa: E402
from oracle import ils_oracle as O  # noqa: E402

GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def g():
    return np.load(os.path.join(GOLD, "golden.npz"))


def _quant_torch(u):
    return torch.floor(torch.clamp(u, 0.0, 1.0) * 255.0 + 0.5).to(torch.uint8)


def test_u8_matches_reference_codec_goldens(g):
    p_rgb = ils.SmoothParams(ils.Charbonnier(0.8, 1e-4), 1.0)
    p_gray = ils.SmoothParams(ils.Welsch(10 / 255), 30.0, iters=10, c=2.0)
    for prec in ("fp64", "fp32"):
        a = ils.smooth_frames_u8(g["u8_rgb_in"], p_rgb, precision=prec)
        b = ils.smooth_frames_u8(g["u8_gray_in"], p_gray, precision=prec)
        assert a.shape == g["u8_rgb_out"].shape and a.dtype == np.uint8
        for got, ref in ((a, g["u8_rgb_out"]), (b, g["u8_gray_out"])):
            d = np.abs(got.astype(int) - ref.astype(int))
            assert d.max() <= 1, prec
            if prec == "fp64":
                assert np.array_equal(got, ref)


def test_u8_path_is_the_float_path_bit_for_bit():
    # fused conversions == converting on the device, smoothing the planes, quantising
    rng = np.random.default_rng(20240607)
    arr = rng.integers(0, 256, size=(2, 1080, 1920, 3), dtype=np.uint8)
    fr = torch.from_numpy(arr).cuda()
    prm = ils.SmoothParams(ils.Charbonnier(0.8, 1e-4), 1.0)
    got = ils.smooth_frames_u8(fr, prm)
    # v / 255 correctly rounded to fp32 (torch's scalar division multiplies by the reciprocal)
    planes = torch.from_numpy((arr.transpose(0, 3, 1, 2).reshape(6, 1080, 1920) / 255.0).astype(np.float32)).cuda()
    u = ils.smooth_batch(planes, prm)
    want = _quant_torch(u).reshape(2, 3, 1080, 1920).permute(0, 2, 3, 1)
    assert torch.equal(got, want)


def test_u8_1080p_matches_oracle():
    rng = np.random.default_rng(7)
    arr = rng.integers(0, 256, size=(1080, 1920, 3), dtype=np.uint8)
    prm = ils.SmoothParams(ils.Charbonnier(0.8, 1e-4), 1.0)
    got = ils.smooth_frames_u8(arr, prm)
    u64 = np.stack([O.smooth_plane(arr[..., k] / 255.0, O.Charbonnier(0.8, 1e-4), 1.0, workers=8)
                    for k in range(3)], axis=-1)
    ref = O.quantize(u64)
    d = np.abs(got.astype(int) - ref.astype(int))
    assert d.max() <= 1
    # a level may differ only where the f64 value sits within the fp32 parity
    # bound (1e-4) of a rounding boundary
    t = np.clip(u64[d != 0], 0.0, 1.0) * 255.0 + 0.5
    assert np.all(np.abs(t - np.rint(t)) <= 255.0 * 1e-4)
    assert (d != 0).mean() < 1e-3


def test_u8_rejects_bad_frames():
    prm = ils.SmoothParams(ils.Charbonnier(0.8, 1e-4), 1.0)
    with pytest.raises(ValueError):
        ils.smooth_frames_u8(np.zeros((8, 8, 3), dtype=np.float32), prm)
    with pytest.raises(ValueError):
        ils.smooth_frames_u8(np.zeros((8, 8, 2), dtype=np.uint8), prm)
    from dataclasses import replace

    with pytest.raises(ValueError):
        ils.smooth_frames_u8(np.zeros((8, 8, 3), dtype=np.uint8), replace(prm, color_mode=ils.ColorMode.LUMINANCE_ONLY))


def test_fused_ingest_equals_planar_path_1080p():
    # 1080p RGB frames take the fused 8-bit ingest (TMA byte rows widened in the
    # first row pass); it must equal smoothing the v/255 planes and quantising
    params = ils.SmoothParams(ils.Charbonnier(0.8, 1e-4), 1.0)
    rng = np.random.default_rng(9)
    f8 = torch.from_numpy(rng.integers(0, 256, (2, 1080, 1920, 3), dtype=np.uint8)).cuda()
    got = ils.smooth_frames_u8(f8, params)
    planes = (f8.permute(0, 3, 1, 2).reshape(6, 1080, 1920).to(torch.float64) / 255.0).to(torch.float32)
    u = ils.smooth_batch(planes, params)
    want = torch.floor(torch.clamp(u, 0, 1) * 255 + 0.5).to(torch.uint8).reshape(2, 3, 1080, 1920).permute(0, 2, 3, 1)
    assert torch.equal(got, want)
