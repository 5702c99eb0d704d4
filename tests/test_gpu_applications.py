"""Application presets on the GPU vs the reference's own outputs.

Goldens: tests/golden/golden.npz app_* (applications.py run by make_golden.py).
Larger sizes against the oracle restatement (pinned in test_oracle_golden.py).
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


def _tol(prec):
    return 1e-10 if prec == "fp64" else 1e-4


@pytest.mark.parametrize("prec", ["fp64", "fp32"])
def test_presets_match_reference_goldens(g, prec):
    img = ils.MultiImage.from_array(g["app_img"])
    prm = ils.SmoothParams(ils.Charbonnier(0.8, 1e-4), 1.0)
    t = _tol(prec)
    out = ils.detail_enhance(img, prm, ils.DetailBoost(3.0), precision=prec).to_array()
    assert np.max(np.abs(out - g["app_detail3"])) < 4 * t  # k = 3 amplifies (f - u) errors
    assert np.max(np.abs(ils.detail_enhance(img, prm, ils.DetailBoost(0.0), precision=prec).to_array()
                         - g["app_detail0"])) < t
    assert np.max(np.abs(ils.clipart_clean(img, 10 / 255, 20.0, precision=prec).to_array() - g["app_clipart"])) < t
    assert np.max(np.abs(ils.texture_smooth(img, 10 / 255, 30.0, 1.0, precision=prec).to_array()
                         - g["app_texture"])) < t
    assert np.max(np.abs(ils.gaussian_blur(img.channels[0], 1.5, precision=prec) - g["app_blur15"])) < t / 100
    assert np.max(np.abs(ils.gaussian_blur(img.channels[1], 0.7, precision=prec) - g["app_blur07"])) < t / 100
    rgb = ils.MultiImage.from_array(g["app_hdr_rgb"], ils.RGB)
    y = ils.luminance(rgb)
    tp = ils.TonemapParams(ils.SmoothParams(ils.Charbonnier(1.0, 1e-4), 2.0), target_range=1.5)
    assert np.max(np.abs(ils.tonemap_single(y, rgb, tp, precision=prec).to_array() - g["app_tm_single"])) < 10 * t
    tpm = ils.TonemapParams(ils.SmoothParams(ils.Charbonnier(1.0, 1e-4), 5.0), lambdas=(0.125, 1.0, 8.0),
                            weights=(1.2, 0.8, 1.0))
    assert np.max(np.abs(ils.tonemap_multi(y, rgb, tpm, precision=prec).to_array() - g["app_tm_multi"])) < 10 * t


def test_detail_enhance_identity_formula_and_constant():
    # test_applications.py:47-84 on the GPU path
    rng = np.random.default_rng(0)
    img = ils.MultiImage.from_array(rng.random((20, 24, 3)))
    prm = ils.SmoothParams(ils.Charbonnier(0.8, 1e-4), 1.0)
    out = ils.detail_enhance(img, prm, ils.DetailBoost(1.0))
    assert all(a.tobytes() == b.tobytes() for a, b in zip(out.channels, img.channels))
    # the fused epilogue is exactly the reference formula applied to our own u (fp64)
    k = 3.0
    out = ils.detail_enhance(img, prm, ils.DetailBoost(k), precision="fp64")
    u = ils.smooth_color(img, prm, precision="fp64")
    for o, f, s in zip(out.channels, img.channels, u.channels):
        assert np.array_equal(o, ils.clip01(s + k * (f - s)))
    const = ils.MultiImage.from_array(np.full((12, 12, 3), 0.42))
    for a in ils.detail_enhance(const, prm, ils.DetailBoost(5.0), precision="fp64").channels:
        assert np.max(np.abs(a - 0.42)) < 1e-11


def test_presets_1080p_match_oracle():
    rng = np.random.default_rng(9)
    arr = rng.random((1080, 1920, 3))
    img = ils.MultiImage.from_array(arr)
    planes = [arr[..., k] for k in range(3)]
    got = ils.texture_smooth(img, 10 / 255, 30.0, 1.0).to_array()
    ref = np.stack(O.texture_smooth(planes, 10 / 255, 30.0, 1.0), -1)
    assert np.max(np.abs(got - ref)) <= 1e-4 and O.psnr(got, ref) >= 60
    got = ils.detail_enhance(img, ils.SmoothParams(ils.Charbonnier(0.8, 1e-4), 1.0), ils.DetailBoost(3.0)).to_array()
    ref = np.stack(O.detail_enhance(planes, O.Charbonnier(0.8, 1e-4), 1.0, 3.0), -1)
    assert np.max(np.abs(got - ref)) <= 4e-4 and O.psnr(got, ref) >= 60


def test_blur_and_tonemap_behaviour():
    # test_applications.py:275-310 / 107-130 on the GPU path
    const = np.full((9, 9), 0.77)
    assert np.max(np.abs(ils.gaussian_blur(const, 2.0) - 0.77)) < 1e-12
    n = 15
    imp = np.zeros((n, n))
    imp[n // 2, n // 2] = 1.0
    x = np.arange(-3, 4, dtype=np.float64)
    k = np.exp(-(x * x) / 2.0)
    k /= k.sum()
    exp = np.zeros((n, n))
    exp[n // 2 - 3: n // 2 + 4, n // 2 - 3: n // 2 + 4] = np.outer(k, k)
    assert np.max(np.abs(ils.gaussian_blur(imp, 1.0) - exp)) < 1e-6
    plane = np.tile(np.linspace(0, 1, 8)[:, None], (1, 6))
    out = ils.gaussian_blur(plane, 1.0)
    assert np.max(np.abs(out - out[:, :1])) < 1e-12
    with pytest.raises(ValueError):
        ils.gaussian_blur(np.zeros((4, 4)), -0.5)
    lum = np.full((16, 16), 7.0)
    tp = ils.TonemapParams(ils.SmoothParams(ils.Charbonnier(1.0, 1e-4), 5.0))
    with pytest.raises(ils.NumericalError):
        ils.tonemap_single(lum, ils.MultiImage((lum, lum, lum), ils.RGB), tp)
    with pytest.raises(ValueError):
        ils.tonemap_single(np.zeros((8, 8)), ils.MultiImage((lum[:8, :8],) * 3, ils.RGB), tp)
    with pytest.raises(ValueError):
        ils.texture_smooth(ils.MultiImage.from_array(np.full((8, 8, 3), 0.5)), 10 / 255, 30.0, sigma_pre=-1.0)


@pytest.mark.parametrize("prec", ["fp32", "fp64"])
def test_tonemap_batched_lambdas_equal_separate_plans(prec):
    # ils_tonemap smooths the three scales as ONE batched launch sequence with a
    # per-plane lambda table; each base must be the smooth of a plan built for
    # its own lambda (applications.py:165-168): rebuild the reference formula
    # (:170-183) on top of three separate smooth_batch calls and compare
    import torch

    rng = np.random.default_rng(12)
    lum = 10.0 ** rng.uniform(-2, 2, (40, 56))
    rgb_planes = tuple(lum * t for t in (0.9, 0.7, 0.5))
    rgb = ils.MultiImage(rgb_planes, ils.RGB)
    base = ils.SmoothParams(ils.Charbonnier(1.0, 1e-4), 5.0)
    tp = ils.TonemapParams(base, lambdas=(0.25, 2.0, 16.0), weights=(1.3, 0.7, 1.1), target_range=1.8)
    got = ils.tonemap_multi(lum, rgb, tp, precision=prec).to_array()
    dt = torch.float32 if prec == "fp32" else torch.float64
    ll = np.log10(lum + tp.log_offset)
    f = torch.from_numpy(ll).to("cuda", dt)[None]
    b = [ils.smooth_batch(f, ils.SmoothParams(base.penalty, lam))[0].double().cpu().numpy() for lam in tp.lambdas]
    spread = b[2].max() - b[2].min()
    out = (b[2] - b[2].max()) * (tp.target_range / spread)
    out = out + tp.weights[2] * (b[1] - b[2]) + tp.weights[1] * (b[0] - b[1]) + tp.weights[0] * (ll - b[0])
    lum_out = 10.0 ** out
    ref = np.stack([np.clip((c / lum) ** tp.saturation * lum_out, 0.0, 1.0) for c in rgb_planes], -1)
    assert np.max(np.abs(got - ref)) < 1e-6  # (GPU vs numpy log10 ulps in the input; a lambda mix-up is ~1e-2)
