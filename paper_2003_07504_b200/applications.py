"""Application presets on the GPU smoother (mirrors reference applications.py:1-222).

Each preset is a batch of smooths plus element-wise work, kept on the device:

* detail_enhance / clipart_clean / texture_smooth: the clip01(u + k (f - u))
  epilogue (k = 0: clip01) is fused into the final row pass of the launch
  sequence (include/ils_b200.h: ils_smooth_epilogue); the channels are one
  batch.
* texture_smooth: the separable replicate-edge Gaussian pre-blur is a CUDA
  kernel pair (ils_gaussian_blur) feeding the smooth without a host trip.
* tonemap_single / tonemap_multi: log10 luminance, the base smooths (the
  three scales of tonemap_multi run concurrently on separate streams), the
  base compression and the recolouring run on the device in float64 around
  the smooths (torch element-wise ops on CUDA tensors; no host arithmetic).

Signatures, defaults, validation and exceptions follow the reference; inputs
and outputs are float64 host MultiImages as there.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, replace

import numpy as np

from . import _lib, _runtime as rt
from .errors import NumericalError
from .image import GRAY, RGB, ColorMode, MultiImage, as_plane
from .penalty import Welsch, is_luminance_only, params_of
from .smoother import SmoothParams, smooth_color


@dataclass(frozen=True)
class DetailBoost:
    """applications.py:23-31: multiplier for the detail layer f - smooth(f); 1 is a no-op."""

    k: float = 3.0

    def __post_init__(self):
        if not (self.k >= 0.0 and np.isfinite(self.k)):
            raise ValueError(f"boost k must be finite and >= 0, got {self.k}")


@dataclass(frozen=True)
class TonemapParams:
    """applications.py:34-77 (same fields, defaults and validation)."""

    base_params: SmoothParams
    target_range: float = 2.0
    saturation: float = 0.6
    log_offset: float = 1e-6
    lambdas: tuple | None = None
    weights: tuple = (1.0, 1.0, 1.0)

    def __post_init__(self):
        if not (self.target_range > 0.0 and np.isfinite(self.target_range)):
            raise ValueError(f"target_range must be finite and positive, got {self.target_range}")
        if not (0.0 < self.saturation <= 1.0):
            raise ValueError(f"saturation must be in (0,1], got {self.saturation}")
        if not (self.log_offset > 0.0 and np.isfinite(self.log_offset)):
            raise ValueError(f"log_offset must be finite and positive, got {self.log_offset}")
        if self.lambdas is not None:
            lams = tuple(float(v) for v in self.lambdas)
            if len(lams) != 3:
                raise ValueError(f"need exactly 3 lambdas, got {len(lams)}")
            if not all(v > 0.0 and np.isfinite(v) for v in lams):
                raise ValueError(f"lambdas must be finite and positive, got {lams}")
            if not (lams[0] <= lams[1] <= lams[2]):
                raise ValueError(f"lambdas must be non-decreasing fine-to-coarse, got {lams}")
            object.__setattr__(self, "lambdas", lams)
        wts = tuple(float(v) for v in self.weights)
        if len(wts) != 3 or not all(np.isfinite(v) for v in wts):
            raise ValueError(f"weights must be 3 finite values, got {self.weights}")
        object.__setattr__(self, "weights", wts)


# ------------------------------------------------------------ device helpers
def _smooth_epilogue(planes, params: SmoothParams, k: float):
    """ILS on CUDA planes [B, H, W] whose last pass writes clip01(u + k (f - u))."""
    torch = rt._torch()
    planes = planes.contiguous()
    B, H, W = planes.shape
    code = _lib.ILS_F32 if planes.dtype == torch.float32 else _lib.ILS_F64
    dev = planes.device
    plan = rt.get_plan(B, H, W, params_of(params), code, dev.index if dev.index is not None else 0)
    out = torch.empty_like(planes)
    ws = torch.empty(plan.workspace_bytes, dtype=torch.uint8, device=dev)
    status = torch.empty(1, dtype=torch.int32, device=dev)
    epi = _lib.Epilogue(_lib.ILS_EPI_DETAIL, float(k))
    _lib.check(_lib.lib().ils_smooth_epilogue(plan.ptr, C.c_void_p(planes.data_ptr()), C.c_void_p(out.data_ptr()),
                                              H * W, C.c_void_p(ws.data_ptr()), rt._stream_ptr(torch, dev),
                                              C.c_void_p(status.data_ptr()), C.byref(epi)), "ils_smooth_epilogue")
    rt.raise_status(int(status.item()))
    return out


def _blur_device(planes, sigma: float):
    """gaussian_blur of CUDA planes [B, H, W] (ils_gaussian_blur)."""
    torch = rt._torch()
    planes = planes.contiguous()
    B, H, W = planes.shape
    out = torch.empty_like(planes)
    tmp = torch.empty_like(planes)
    code = _lib.ILS_F32 if planes.dtype == torch.float32 else _lib.ILS_F64
    _lib.check(_lib.lib().ils_gaussian_blur(C.c_void_p(planes.data_ptr()), C.c_void_p(out.data_ptr()),
                                            C.c_void_p(tmp.data_ptr()), B, H, W, H * W, float(sigma), code,
                                            rt._stream_ptr(torch, planes.device)), "ils_gaussian_blur")
    return out


def _image_out(planes, space):
    return MultiImage(tuple(rt.to_host_f64(planes)), space)


# ------------------------------------------------------------ presets
def detail_enhance(img: MultiImage, params: SmoothParams, boost: DetailBoost = DetailBoost(), *,
                   precision: str | None = None) -> MultiImage:
    """applications.py:80-93: clip01(u + k (f - u)); k = 1 returns the input as-is."""
    if boost.k == 1.0:
        return img
    if is_luminance_only(params) and img.space == RGB:
        # u comes from the YUV round trip (smooth_color on the GPU); the boost
        # is element-wise on the device in float64
        torch = rt._torch()
        u = smooth_color(img, params, precision=precision)
        f = torch.tensor(np.stack(img.channels), device="cuda")
        s = torch.tensor(np.stack(u.channels), device="cuda")
        out = torch.clamp(s + boost.k * (f - s), 0.0, 1.0)
        return _image_out(out, img.space)
    planes = rt.to_device_planes(img.channels, precision)
    return _image_out(_smooth_epilogue(planes, params, boost.k), img.space)


def _check_hdr_inputs(lum, rgb: MultiImage) -> None:
    """applications.py:96-108."""
    if rgb.space != RGB:
        raise ValueError(f"tone mapping needs an rgb image, got {rgb.space!r}")
    if lum.shape != (rgb.height, rgb.width):
        raise ValueError(f"luminance {lum.shape} does not match image {(rgb.height, rgb.width)}")
    if not np.all(lum > 0.0):
        raise ValueError("hdr luminance must be strictly positive")
    for ch in rgb.channels:
        if not np.all(ch >= 0.0):
            raise ValueError("hdr rgb channels must be non-negative")


def _compress_base(base, target_range: float):
    """applications.py:111-118 on a CUDA float64 tensor."""
    spread = float(base.max() - base.min())
    if spread < 1e-9:
        raise NumericalError(f"degenerate base dynamic range {spread:g}; nothing to compress")
    cf = target_range / spread
    return (base - base.max()) * cf


def _recolor(lum, rgb_planes, log_lum_out, saturation: float) -> MultiImage:
    """applications.py:121-129 on CUDA float64 tensors."""
    torch = rt._torch()
    lum_out = torch.pow(10.0, log_lum_out)
    out = torch.clamp(torch.pow(rgb_planes / lum, saturation) * lum_out, 0.0, 1.0)
    return _image_out(out, RGB)


def _bases(log_lum64, params_list, precision):
    """Smooth the log luminance once per parameter set; the sets run concurrently on separate streams."""
    torch = rt._torch()
    dt = rt.torch_dtype(precision)
    f = log_lum64.to(dt)[None]
    cur = torch.cuda.current_stream()
    outs = [None] * len(params_list)
    streams = [torch.cuda.Stream() for _ in params_list]
    statuses = []
    for i, (prm, st) in enumerate(zip(params_list, streams)):
        st.wait_stream(cur)
        with torch.cuda.stream(st):
            u, _, status = rt.smooth_device(f, params_of(prm), check=False)
            outs[i] = u[0]
            statuses.append(status)
    for st in streams:
        cur.wait_stream(st)
    for u in outs:
        u.record_stream(cur)
    for s in statuses:
        rt.raise_status(int(s.item()))
    return [u.to(torch.float64) for u in outs]


def tonemap_single(hdr_luminance, rgb: MultiImage, tp: TonemapParams, *, precision: str | None = None) -> MultiImage:
    """applications.py:132-150."""
    torch = rt._torch()
    lum = as_plane(hdr_luminance)
    _check_hdr_inputs(lum, rgb)
    lum_d = torch.tensor(lum, device="cuda")
    log_lum = torch.log10(lum_d + tp.log_offset)
    (base,) = _bases(log_lum, [tp.base_params], precision)
    detail = log_lum - base
    log_lum_out = _compress_base(base, tp.target_range) + detail
    return _recolor(lum_d, torch.tensor(np.stack(rgb.channels), device="cuda"), log_lum_out, tp.saturation)


def tonemap_multi(hdr_luminance, rgb: MultiImage, tp: TonemapParams, *, precision: str | None = None) -> MultiImage:
    """applications.py:153-183: three scales, coarsest base compressed, details reweighted."""
    if tp.lambdas is None:
        raise ValueError("tonemap_multi needs tp.lambdas (a fine-to-coarse triple)")
    torch = rt._torch()
    lum = as_plane(hdr_luminance)
    _check_hdr_inputs(lum, rgb)
    lum_d = torch.tensor(lum, device="cuda")
    log_lum = torch.log10(lum_d + tp.log_offset)
    b = _bases(log_lum, [replace(tp.base_params, lam=lam) for lam in tp.lambdas], precision)
    d0 = log_lum - b[0]
    d1 = b[0] - b[1]
    d2 = b[1] - b[2]
    w0, w1, w2 = tp.weights
    log_lum_out = _compress_base(b[2], tp.target_range) + w2 * d2 + w1 * d1 + w0 * d0
    return _recolor(lum_d, torch.tensor(np.stack(rgb.channels), device="cuda"), log_lum_out, tp.saturation)


def clipart_clean(img: MultiImage, gamma: float, lam: float, *, precision: str | None = None) -> MultiImage:
    """applications.py:186-197: Welsch, c = 2, 10 iterations, per channel, clip01 (fused)."""
    params = SmoothParams(Welsch(gamma), lam, iters=10, c=2.0, color_mode=ColorMode.PER_CHANNEL_RGB)
    planes = rt.to_device_planes(img.channels, precision)
    return _image_out(_smooth_epilogue(planes, params, 0.0), img.space)


def texture_smooth(img: MultiImage, gamma: float, lam: float, sigma_pre: float = 1.0, *,
                   precision: str | None = None) -> MultiImage:
    """applications.py:200-207: Gaussian pre-blur, Welsch 15 iterations, clip01 -- all on the device."""
    if not (sigma_pre >= 0.0 and np.isfinite(sigma_pre)):
        raise ValueError(f"sigma_pre must be finite and >= 0, got {sigma_pre}")
    params = SmoothParams(Welsch(gamma), lam, iters=15, color_mode=ColorMode.PER_CHANNEL_RGB)
    planes = rt.to_device_planes(img.channels, precision)
    if sigma_pre > 0.0:
        planes = _blur_device(planes, sigma_pre)
    return _image_out(_smooth_epilogue(planes, params, 0.0), img.space)


def gaussian_blur(plane, sigma: float, *, precision: str | None = "fp64"):
    """applications.py:210-222: separable Gaussian, radius ceil(3 sigma), replicate edges."""
    plane = as_plane(plane)
    if not (sigma >= 0.0 and np.isfinite(sigma)):
        raise ValueError(f"sigma must be finite and >= 0, got {sigma}")
    if sigma == 0.0:
        return np.array(plane)
    return rt.to_host_f64(_blur_device(rt.to_device_planes([plane], precision), sigma))[0]


__all__ = ["DetailBoost", "TonemapParams", "clipart_clean", "detail_enhance", "gaussian_blur", "texture_smooth",
           "tonemap_multi", "tonemap_single", "GRAY"]
