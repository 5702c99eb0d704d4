"""Penalty parameter objects of the drop-in (mirrors reference penalty.py:40-126).

These carry the parameters (validated exactly as the reference does) and the
closed-form min_curvature the smoother needs.  value/derivative/edge_stop are
host-side scalar/array helpers kept for API parity; the smoothing path never
calls them -- phi'(x) and mu = c x - phi'(x) are evaluated inside the fused
CUDA row kernel (csrc/ils_kernels.cuh: dphi/aux).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

DEFAULT_EPS = 1e-4
_CURVATURE_SLACK = 1e-12


@dataclass(frozen=True)
class Charbonnier:
    """Generalized Charbonnier penalty (x^2 + eps)^(p/2) (penalty.py:47-75)."""

    p: float = 0.8
    eps: float = DEFAULT_EPS

    def __post_init__(self):
        if not (0.0 < self.p <= 1.0):
            raise ValueError("p must be in (0,1]")
        if not (self.eps > 0.0):
            raise ValueError(f"eps must be positive, got {self.eps}")

    def value(self, x):
        x = np.asarray(x, dtype=np.float64)
        return (x * x + self.eps) ** (self.p / 2.0)

    def derivative(self, x):
        x = np.asarray(x, dtype=np.float64)
        return self.p * x * (x * x + self.eps) ** (self.p / 2.0 - 1.0)

    def edge_stop(self, x):
        x = np.asarray(x, dtype=np.float64)
        return (self.p / 2.0) * (x * x + self.eps) ** (self.p / 2.0 - 1.0)

    @property
    def min_curvature(self) -> float:
        return self.p * self.eps ** (self.p / 2.0 - 1.0)


@dataclass(frozen=True)
class Welsch:
    """Welsch penalty 2 g^2 (1 - exp(-x^2 / 2 g^2)) (penalty.py:78-105)."""

    gamma: float

    def __post_init__(self):
        if not (self.gamma > 0.0):
            raise ValueError(f"gamma must be positive, got {self.gamma}")

    def value(self, x):
        x = np.asarray(x, dtype=np.float64)
        g2 = self.gamma * self.gamma
        return 2.0 * g2 * (1.0 - np.exp(-x * x / (2.0 * g2)))

    def derivative(self, x):
        x = np.asarray(x, dtype=np.float64)
        g2 = self.gamma * self.gamma
        return 2.0 * x * np.exp(-x * x / (2.0 * g2))

    def edge_stop(self, x):
        x = np.asarray(x, dtype=np.float64)
        g2 = self.gamma * self.gamma
        return np.exp(-x * x / (2.0 * g2))

    @property
    def min_curvature(self) -> float:
        return 2.0


def check_curvature(spec, c: float) -> None:
    """penalty.py:108-114."""
    c0 = spec.min_curvature
    if not np.isfinite(c) or c < c0 * (1.0 - _CURVATURE_SLACK):
        raise ValueError(
            f"curvature c={c} is below the minimum {c0} required for a "
            f"convex bound with {type(spec).__name__}"
        )


def aux_update(spec, c: float, x):
    """Optimal auxiliary variable c x - phi'(x), elementwise (penalty.py:117-126), on the GPU.

    numpy in -> float64 numpy out; a CUDA tensor -> tensor of the same dtype.
    """
    check_curvature(spec, c)
    from . import _runtime as rt

    return rt.aux_fields(to_c_params(spec, 1.0, float(c), 1), x)


def soft_threshold(x, alpha: float):
    """penalty.py:168-177 (host helper; the HQS field step runs fused in the row kernel)."""
    if not (alpha >= 0.0 and np.isfinite(alpha)):
        raise ValueError(f"alpha must be finite and >= 0, got {alpha}")
    x = np.asarray(x, dtype=np.float64)
    return np.where(np.abs(x) <= alpha, 0.0, x - alpha * np.sign(x))


def huber(x, alpha: float):
    """penalty.py:180-191 (host helper)."""
    if not (alpha > 0.0 and np.isfinite(alpha)):
        raise ValueError(f"alpha must be finite and > 0, got {alpha}")
    x = np.asarray(x, dtype=np.float64)
    return np.where(np.abs(x) <= alpha, x * x / (2.0 * alpha), np.abs(x) - alpha / 2.0)


def penalty_kind(spec) -> str:
    """'charbonnier' / 'welsch' for this package's penalties and for any object
    with the reference's fields (the reference's own frozen dataclasses,
    penalty.py:47-105), so reference parameter objects can be passed straight in."""
    if isinstance(spec, Charbonnier):
        return "charbonnier"
    if isinstance(spec, Welsch):
        return "welsch"
    name = type(spec).__name__
    if name == "Charbonnier" or (hasattr(spec, "p") and hasattr(spec, "eps") and not hasattr(spec, "gamma")):
        return "charbonnier"
    if name == "Welsch" or (hasattr(spec, "gamma") and not hasattr(spec, "p")):
        return "welsch"
    raise ValueError(f"unsupported penalty {name}: the CUDA path implements Charbonnier and Welsch")


def to_c_params(spec, lam: float, c: float, iters: int):
    """Flatten (penalty, lam, c, iters) into the C ABI's ils_params."""
    from ._lib import ILS_CHARBONNIER, ILS_WELSCH, Params

    if penalty_kind(spec) == "charbonnier":
        return Params(ILS_CHARBONNIER, float(spec.p), float(spec.eps), 0.0, float(lam), float(c), int(iters))
    return Params(ILS_WELSCH, 0.0, 0.0, float(spec.gamma), float(lam), float(c), int(iters))


def params_of(params):
    """ils_params of a SmoothParams -- this package's or the reference's
    (smoother.py:31-62: .penalty, .lam, .iters, .c / .curvature)."""
    c = getattr(params, "curvature", None)
    if c is None:
        c = params.penalty.min_curvature if params.c is None else float(params.c)
    return to_c_params(params.penalty, params.lam, float(c), params.iters)


def is_luminance_only(params) -> bool:
    """ColorMode.LUMINANCE_ONLY of either package's enum (compared by value)."""
    mode = getattr(params, "color_mode", None)
    return getattr(mode, "value", mode) == "luminance_only"
