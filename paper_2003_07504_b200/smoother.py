"""ILS smoothing entry points of the drop-in (mirrors reference smoother.py:31-217).

smooth_plane / smooth_color keep the reference's signatures, defaults,
validation, return types and exceptions.  All iterations of a call run on
the GPU as one launch sequence (ils_smooth): iteration 0 row pass from f,
then per iteration a column pass and a fused row pass, then a final row
pass writing u.  Channels (and, via smooth_batch, frames) are a batch
dimension of that single sequence instead of a thread pool
(smoother.py:205-210).  `workers` is validated and accepted but cannot
change results: one GPU launch does the work.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import _runtime as rt
from .image import GRAY, RGB, YUV, ColorMode, MultiImage, as_plane
from .penalty import is_luminance_only, params_of, to_c_params
from .solver import SolverPlan, make_plan


@dataclass(frozen=True)
class SmoothParams:
    """Settings for one smoothing run (smoother.py:31-62)."""

    penalty: object
    lam: float
    iters: int = 4
    c: float | None = None
    color_mode: ColorMode = ColorMode.PER_CHANNEL_RGB

    def __post_init__(self):
        if not (self.lam > 0.0 and np.isfinite(self.lam)):
            raise ValueError(f"lam must be finite and positive, got {self.lam}")
        if not (isinstance(self.iters, int) and self.iters >= 1):
            raise ValueError(f"iters must be an integer >= 1, got {self.iters}")
        if self.c is not None:
            c0 = self.penalty.min_curvature
            if not np.isfinite(self.c) or self.c < c0 * (1.0 - 1e-12):
                raise ValueError(f"c={self.c} is below the penalty's minimum curvature {c0}")
        if not isinstance(self.color_mode, ColorMode):
            raise ValueError(f"color_mode must be a ColorMode, got {self.color_mode!r}")

    @property
    def curvature(self) -> float:
        return self.penalty.min_curvature if self.c is None else float(self.c)

    def c_params(self):
        return to_c_params(self.penalty, self.lam, self.curvature, self.iters)


@dataclass
class EnergyTrace:
    """Objective values per iteration; energies[0] is E at the input (smoother.py:65-90)."""

    energies: list = field(default_factory=list)

    def __len__(self) -> int:
        return len(self.energies)

    def rel_decrease(self, n: int, reference: float | None = None) -> float:
        if not self.energies:
            raise ValueError("empty trace")
        if not (0 <= n < len(self.energies)):
            raise ValueError(f"iteration {n} outside trace of length {len(self.energies)}")
        e0 = self.energies[0]
        ref = self.energies[-1] if reference is None else float(reference)
        den = e0 - ref
        if den == 0.0:
            return 1.0
        return (e0 - self.energies[n]) / den


def energy(u, f, penalty, lam: float) -> float:
    """Objective value: data term plus penalized periodic gradients (smoother.py:93-101), on the GPU.

    Deterministic f64 reduction; 2-D inputs return a float, stacked CUDA
    tensors [B, H, W] a float64 tensor [B].
    """
    if tuple(np.shape(u)) != tuple(np.shape(f)):
        raise ValueError(f"shapes differ: u {tuple(np.shape(u))}, f {tuple(np.shape(f))}")
    return rt.energy_fields(to_c_params(penalty, float(lam), penalty.min_curvature, 1), u, f)


def _is_tensor(x) -> bool:
    try:
        import torch
    except ImportError:  # pragma: no cover
        return False
    return isinstance(x, torch.Tensor)


def smooth_batch(f, params: SmoothParams, trace: bool = False):
    """Smooth a CUDA tensor of planes f[B, H, W] (channels x frames) in one launch.

    Returns u[B, H, W] (same dtype/device) or (u, energies[(iters+1), B]).
    """
    u, energies, _ = rt.smooth_device(f, params_of(params), trace=trace, check=True)
    return (u, energies) if trace else u


def smooth_frames_u8(frames, params: SmoothParams, *, precision: str | None = None):
    """8-bit frames through the fused ingest/egress path.

    frames: uint8 [F, H, W, C], [H, W, C] or [H, W] (numpy or CUDA tensor;
    C = 3 rgb or 1 gray, the PNG/PPM pixel layout of formats.py).  Returns
    the same shape and kind: floor(clip01(u) * 255 + 0.5) of smooth_color on
    the planes v / 255 (formats.py:25-27 + smoother.py:175-217), per channel.
    """
    if is_luminance_only(params):
        raise ValueError("the 8-bit path smooths channels independently (PER_CHANNEL_RGB or gray)")
    torch = rt._torch()
    is_t = _is_tensor(frames)
    t = frames if is_t else torch.from_numpy(np.ascontiguousarray(frames))
    if t.dtype != torch.uint8:
        raise ValueError(f"8-bit path expects uint8 frames, got {t.dtype}")
    shape = tuple(t.shape)
    if len(shape) == 2:
        t4 = t.reshape(1, shape[0], shape[1], 1)
    elif len(shape) == 3:
        t4 = t.unsqueeze(0)
    elif len(shape) == 4:
        t4 = t
    else:
        raise ValueError(f"frames must be [H, W], [H, W, C] or [F, H, W, C], got {shape}")
    if t4.shape[-1] not in (1, 3):
        raise ValueError(f"expected 1 or 3 channels, got {t4.shape[-1]}")
    if t4.numel() == 0:
        raise ValueError("image plane must be non-empty")
    u = rt.smooth_device_u8(t4.to("cuda") if not t4.is_cuda else t4, params_of(params), precision)
    u = u.reshape(shape)
    return u if (is_t and frames.is_cuda) else u.cpu().numpy()


def _check_plan(plan: SolverPlan, shape, params: SmoothParams):
    """smoother.py:149-159."""
    if (plan.height, plan.width) != tuple(shape):
        raise ValueError(f"plan is {plan.height}x{plan.width}, plane is {tuple(shape)}")
    if plan.lam != params.lam or plan.c != params.curvature:
        raise ValueError("plan was built for different lam or c")


def smooth_plane(f, params: SmoothParams, trace: bool = False, plan: SolverPlan | None = None, workers: int = 1,
                 *, precision: str | None = None):
    """Smooth one plane (smoother.py:132-172). Returns u or (u, EnergyTrace).

    numpy/array-like input -> float64 numpy output (reference semantics);
    a CUDA tensor [H, W] -> CUDA tensor of the same dtype, zero-copy.
    """
    if workers < 1:
        raise ValueError(f"workers must be >= 1, got {workers}")
    if _is_tensor(f):
        if f.dim() != 2:
            raise ValueError(f"image plane must be 2-D, got shape {tuple(f.shape)}")
        if plan is not None:
            _check_plan(plan, f.shape, params)
        u, en, _ = rt.smooth_device(f.unsqueeze(0), params_of(params), trace=trace, check=True)
        if trace:
            return u[0], EnergyTrace([float(v) for v in en[:, 0].tolist()])
        return u[0]
    f = as_plane(f)
    if plan is not None:
        _check_plan(plan, f.shape, params)
    dev = rt.to_device_planes([f], precision)
    u, en, _ = rt.smooth_device(dev, params_of(params), trace=trace, check=True)
    out = rt.to_host_f64(u)[0]
    if trace:
        return out, EnergyTrace([float(v) for v in en[:, 0].tolist()])
    return out


def _image_like(img, channels, space):
    """The result image in the caller's MultiImage type (this package's, or the
    reference's when its objects are passed in after a monkeypatch)."""
    if isinstance(img, MultiImage):
        return MultiImage._trusted(tuple(channels), space)
    return type(img)(tuple(channels), space)


def smooth_color(img: MultiImage, params: SmoothParams, trace: bool = False, workers: int = 1,
                 *, precision: str | None = None):
    """Smooth a gray or RGB image (smoother.py:175-217). Returns image or (image, trace).

    PER_CHANNEL_RGB: the channels are staged, smoothed and returned plane by
    plane in a pipeline (rt.smooth_planes_host); with trace=True they are one
    batch of one launch sequence and the energies are summed over channels
    in channel order.
    LUMINANCE_ONLY: BT.601 conversion, Y smoothed, inverse conversion, all on
    the GPU.  Output is not clipped.
    """
    if workers < 1:
        raise ValueError(f"workers must be >= 1, got {workers}")
    if img.space == YUV:
        raise ValueError("smooth_color expects a gray or rgb image")
    if img.space == GRAY:
        res = smooth_plane(img.channels[0], params, trace, workers=workers, precision=precision)
        if trace:
            return _image_like(img, (res[0],), GRAY), res[1]
        return _image_like(img, (res,), GRAY)
    cp = params_of(params)
    if not trace and not is_luminance_only(params):
        # the channels are independent (smoother.py:204-213): staged, smoothed
        # and returned plane by plane in a pipeline (same bits as the batch)
        res = rt.smooth_planes_host(img.channels, cp, precision)
        if res is not None:
            return _image_like(img, res, RGB)
    planes = rt.to_device_planes(img.channels, precision)
    if is_luminance_only(params):
        rt.rgb_yuv_(planes, inverse=False)
        u, en, _ = rt.smooth_device(planes[0:1], cp, trace=trace, check=True)
        planes[0:1] = u
        rt.rgb_yuv_(planes, inverse=True)
        out = _image_like(img, rt.to_host_f64(planes), RGB)
        if trace:
            return out, EnergyTrace([float(v) for v in en[:, 0].tolist()])
        return out
    u, en, _ = rt.smooth_device(planes, cp, trace=trace, check=True)
    out = _image_like(img, rt.to_host_f64(u), RGB)
    if trace:
        summed = [float(sum(row)) for row in en.tolist()]
        return out, EnergyTrace(summed)
    return out
