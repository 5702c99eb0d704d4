"""Spectral least-squares solve of the drop-in (mirrors reference solver.py:52-134).

make_plan/SolverPlan keep the reference's signature and validation; the
arithmetic (r2c row FFT, column FFT, / denom, inverse column FFT, c2r) runs
in libils_b200.so.  The smoothing kernels never materialise the denominator
as an H x W array (they evaluate 1 + c lam/2 (wy[ky] + wx[kx]) from two 1-D
tables) and never form F(f) (f is added in the spatial domain); the plan's
`denom` and `f_hat` fields are still the reference's arrays, computed on the
GPU, for callers that read them (e.g. hqs.py:53).
"""

from __future__ import annotations

from dataclasses import dataclass, replace

import numpy as np

from . import _runtime as rt
from .penalty import Welsch, to_c_params


@dataclass(frozen=True, eq=False)
class SolverPlan:
    """Per-(shape, lam, c) plan (solver.py:52-75), same fields in the same order.

    denom is the H x W float64 spectral denominator and f_hat, once
    with_data ran, the complex128 fft2 of the data plane -- both computed on
    the GPU (the hand-written transforms) and returned as numpy arrays, as the
    reference holds them.  The CUDA smoothing path needs neither: it
    evaluates the denominator from two 1-D tables inside the column pass and
    adds f in the spatial domain (F(f) is never formed).
    """

    height: int
    width: int
    lam: float
    c: float
    denom: object = None
    f_hat: object = None
    workers: int = 1

    def with_data(self, f) -> "SolverPlan":
        """Return a copy of the plan with f's transform cached (solver.py:69-75)."""
        f = np.asarray(f)
        if f.shape != (self.height, self.width):
            raise ValueError(f"plan is {self.height}x{self.width}, data is {f.shape}")
        return replace(self, f_hat=rt.fft2_full(f))


def make_plan(height: int, width: int, lam: float, c: float, f=None, workers: int = 1) -> SolverPlan:
    """solver.py:78-106: validation, then the analytic denominator (on the GPU)."""
    if height < 1 or width < 1:
        raise ValueError(f"invalid plan size {height}x{width}")
    if not (lam > 0.0 and np.isfinite(lam)):
        raise ValueError(f"lam must be finite and positive, got {lam}")
    if not (c > 0.0 and np.isfinite(c)):
        raise ValueError(f"c must be finite and positive, got {c}")
    if workers < 1:
        raise ValueError(f"workers must be >= 1, got {workers}")
    plan = SolverPlan(int(height), int(width), float(lam), float(c), rt.denominator(height, width, lam, c), None,
                      int(workers))
    if f is not None:
        plan = plan.with_data(f)
    return plan


def solve_ls(plan: SolverPlan, f, mu_x, mu_y, *, precision=None):
    """u = argmin of the quadratic bound energy (solver.py:109-134), on the GPU.

    numpy inputs return a float64 numpy array (C-contiguous, like the
    reference), computed in float64 unless precision="fp32"; CUDA tensors
    [H, W] or [B, H, W] (f, mu_x, mu_y of one shape, dtype and device) return
    a CUDA tensor of that dtype.
    """
    import torch

    shape = (plan.height, plan.width)
    is_t = isinstance(f, torch.Tensor)
    arrs = (("f", f), ("mu_x", mu_x), ("mu_y", mu_y))
    for name, a in arrs:
        shp = tuple(a.shape[-2:]) if is_t else np.shape(a)
        if shp != shape:
            raise ValueError(f"{name} has shape {tuple(np.shape(a))}, plan expects {shape}")
    # solve_ls takes (lam, c) from the plan; the penalty slot is unused.
    cp = to_c_params(Welsch(1.0), plan.lam, plan.c, 1)
    if is_t:
        for name, a in arrs[1:]:
            if not isinstance(a, torch.Tensor) or a.shape != f.shape or a.dtype != f.dtype or a.device != f.device:
                raise ValueError(f"{name} must be a tensor of f's shape {tuple(f.shape)}, dtype {f.dtype} and "
                                 f"device {f.device}")
        if f.dim() not in (2, 3):
            raise ValueError(f"f must be [H, W] or [B, H, W], got shape {tuple(f.shape)}")
        t = [a if a.dim() == 3 else a.unsqueeze(0) for _, a in arrs]
        u = rt.solve_device(*t, cp)
        return u if f.dim() == 3 else u[0]
    # one staging copy for the three planes (they share the pinned buffer)
    prec = precision or "fp64"
    if precision is None and not rt.plan_supported(plan.height, plan.width, "fp64"):
        prec = "fp32"  # fp64 lines stop at about 4096 points: such planes solve in fp32
    dev = rt.to_device_planes([np.asarray(a, dtype=np.float64) for _, a in arrs], prec)
    u = rt.solve_device(dev[0:1], dev[1:2], dev[2:3], cp)
    return rt.to_host_f64(u)[0]


def grad_x(u):
    """Forward difference along axis 1, wrapping at the right edge (solver.py:33-35), on the GPU.

    numpy in -> float64 numpy out (bit-identical to the reference); a CUDA
    tensor [H, W] or [B, H, W] -> tensor of the same dtype.
    """
    return rt.grad_fields(u, "x")


def grad_y(u):
    """Forward difference along axis 0, wrapping at the bottom edge (solver.py:38-40), on the GPU."""
    return rt.grad_fields(u, "y")


def adjoint_accumulate(mu_x, mu_y):
    """Sum of the adjoints of grad_x and grad_y applied to a field pair (solver.py:43-49), on the GPU."""
    return rt.adjoint_fields(mu_x, mu_y)
