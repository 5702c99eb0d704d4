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
        f = torch.from_numpy(np.stack(img.channels)).to("cuda")
        s = torch.from_numpy(np.stack(u.channels)).to("cuda")
        out = torch.empty_like(f)
        _lib.check(_lib.lib().ils_detail_boost(C.c_void_p(f.data_ptr()), C.c_void_p(s.data_ptr()),
                                               C.c_void_p(out.data_ptr()), f.numel(), float(boost.k), _lib.ILS_F64,
                                               rt._stream_ptr(torch, f.device)), "ils_detail_boost")
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


def _tonemap(hdr_luminance, rgb: MultiImage, tp: TonemapParams, lambdas, precision) -> MultiImage:
    """applications.py:132-183 through ils_tonemap: log10 luminance, every scale's base
    smoothing in one batched launch sequence (a lambda per plane), base compression and
    recolouring -- all hand-written kernels, float64 in and out."""
    torch = rt._torch()
    lum = as_plane(hdr_luminance)
    _check_hdr_inputs(lum, rgb)
    ns = len(lambdas)
    prm = tp.base_params
    code = _lib.ILS_F32 if (precision or rt.get_default_precision()) == "fp32" else _lib.ILS_F64
    H, W = lum.shape
    plan = rt.get_plan(ns, H, W, params_of(replace(prm, lam=float(lambdas[-1]))), code, torch.cuda.current_device())
    c = _lib.TonemapParamsC()
    c.nscales = ns
    for k in range(3):
        c.lam[k] = float(lambdas[min(k, ns - 1)])
        c.weights[k] = float(tp.weights[k])
    c.target_range, c.saturation, c.log_offset = float(tp.target_range), float(tp.saturation), float(tp.log_offset)
    L = _lib.lib()
    wsz = C.c_size_t()
    _lib.check(L.ils_tonemap_workspace_size(plan.ptr, C.byref(wsz)), "ils_tonemap_workspace_size")
    lum_d = torch.from_numpy(np.ascontiguousarray(lum)).to("cuda")
    rgb_d = torch.from_numpy(np.ascontiguousarray(np.stack(rgb.channels))).to("cuda")
    out = torch.empty_like(rgb_d)
    ws = torch.empty(wsz.value, dtype=torch.uint8, device="cuda")
    status = torch.empty(1, dtype=torch.int32, device="cuda")
    sc = torch.empty(3, dtype=torch.float64, device="cuda")
    _lib.check(L.ils_tonemap(plan.ptr, C.c_void_p(lum_d.data_ptr()), C.c_void_p(rgb_d.data_ptr()),
                             C.c_void_p(out.data_ptr()), C.byref(c), C.c_void_p(ws.data_ptr()),
                             rt._stream_ptr(torch, lum_d.device), C.c_void_p(status.data_ptr()),
                             C.c_void_p(sc.data_ptr())), "ils_tonemap")
    rt.raise_status(int(status.item()))
    spread = float(sc[1].item())
    if spread < 1e-9:  # _compress_base, applications.py:112-116
        raise NumericalError(f"degenerate base dynamic range {spread:g}; nothing to compress")
    return _image_out(out, RGB)


def tonemap_single(hdr_luminance, rgb: MultiImage, tp: TonemapParams, *, precision: str | None = None) -> MultiImage:
    """applications.py:132-150 (one scale: base, detail, compression, recolouring)."""
    return _tonemap(hdr_luminance, rgb, tp, (tp.base_params.lam,), precision)


def tonemap_multi(hdr_luminance, rgb: MultiImage, tp: TonemapParams, *, precision: str | None = None) -> MultiImage:
    """applications.py:153-183: three scales, coarsest base compressed, details reweighted."""
    if tp.lambdas is None:
        raise ValueError("tonemap_multi needs tp.lambdas (a fine-to-coarse triple)")
    return _tonemap(hdr_luminance, rgb, tp, tp.lambdas, precision)


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
