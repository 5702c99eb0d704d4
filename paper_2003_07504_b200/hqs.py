"""Penalty-splitting (HQS) baseline of the drop-in (mirrors reference hqs.py:1-66).

Minimises sum (u - f)^2 + lam sum_d |grad_d u| by alternating the field step
m = soft_threshold(grad u, alpha_n), alpha_n = lam / (2 beta_n), with the
u-step solve_ls(lam = 2 beta_n, c = 1), beta_n = beta0 kappa^n.

On the GPU this is the ILS launch sequence with per-iteration parameters
(include/ils_b200.h: ils_hqs_plan_create): the soft threshold is fused into
the row pass exactly where the ILS stencil evaluates mu = c x - phi'(x), and
the column pass evaluates the per-iteration denominator 1 + beta_n (wy + wx)
analytically, so one plan serves every beta_n of the schedule.  As in the
reference (hqs.py:51-53) the data transform is iteration independent: f is
added in the spatial domain before each forward transform.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib, _runtime as rt
from .image import as_plane


@dataclass(frozen=True)
class HqsParams:
    """hqs.py:27-47 (same fields, defaults and validation messages)."""

    lam: float
    beta0: float | None = None  # None: 2 * lam
    kappa: float = 2.0
    iters: int = 4

    def __post_init__(self):
        if not (self.lam > 0.0 and np.isfinite(self.lam)):
            raise ValueError(f"lam must be finite and positive, got {self.lam}")
        if self.beta0 is not None and not (self.beta0 > 0.0 and np.isfinite(self.beta0)):
            raise ValueError(f"beta0 must be finite and positive, got {self.beta0}")
        if not (self.kappa > 1.0 and np.isfinite(self.kappa)):
            raise ValueError(f"kappa must be finite and > 1, got {self.kappa}")
        if not (isinstance(self.iters, int) and self.iters >= 1):
            raise ValueError(f"iters must be an integer >= 1, got {self.iters}")

    @property
    def initial_beta(self) -> float:
        return 2.0 * self.lam if self.beta0 is None else float(self.beta0)

    def c_params(self):
        """The C ABI's ils_hqs_params."""
        return _lib.HqsParams(float(self.lam), float(self.initial_beta), float(self.kappa), int(self.iters))


def hqs_smooth_plane(f, params: HqsParams, workers: int = 1, *, precision: str | None = None):
    """hqs.py:50-66.  numpy in -> float64 numpy out; a CUDA tensor [H, W] -> CUDA tensor.

    Raises NumericalError naming the first iteration whose iterate is not
    finite (hqs.py:64-65), ValueError for a non-finite input plane.
    """
    if workers < 1:
        raise ValueError(f"workers must be >= 1, got {workers}")
    from .smoother import _is_tensor

    if _is_tensor(f):
        if f.dim() != 2:
            raise ValueError(f"image plane must be 2-D, got shape {tuple(f.shape)}")
        u, _, _ = rt.smooth_device(f.unsqueeze(0), params.c_params(), check=True)
        return u[0]
    f = as_plane(f)
    dev = rt.to_device_planes([f], precision)
    u, _, _ = rt.smooth_device(dev, params.c_params(), check=True)
    return rt.to_host_f64(u)[0]


def hqs_smooth_batch(f, params: HqsParams):
    """All planes of a CUDA tensor [..., H, W] in one launch sequence (the CLI's per-channel loop, cli.py:257-263)."""
    shape = f.shape
    u, _, _ = rt.smooth_device(f.reshape(-1, shape[-2], shape[-1]), params.c_params(), check=True)
    return u.reshape(shape)
