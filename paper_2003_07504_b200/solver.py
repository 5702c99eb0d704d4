"""Spectral least-squares solve of the drop-in (mirrors reference solver.py:52-134).

make_plan/SolverPlan keep the reference's signature and validation; the
arithmetic (r2c row FFT, column FFT, / denom, inverse column FFT, c2r) runs
in libils_b200.so.  The denominator is never materialised as an H x W array:
the kernels evaluate 1 + c lam/2 (wy[ky] + wx[kx]) from two 1-D tables, so
`denom` is not a field here.  F(f) is not cached either -- the CUDA path adds
f in the spatial domain -- so with_data only validates and records f.
"""

from __future__ import annotations

from dataclasses import dataclass, replace

import numpy as np

from . import _runtime as rt
from .penalty import Welsch, to_c_params


@dataclass(frozen=True, eq=False)
class SolverPlan:
    """Per-(shape, lam, c) plan (solver.py:52-75)."""

    height: int
    width: int
    lam: float
    c: float
    f_hat: object = None  # the bound data plane (with_data); kept for API parity
    workers: int = 1

    def with_data(self, f) -> "SolverPlan":
        f = np.asarray(f)
        if f.shape != (self.height, self.width):
            raise ValueError(f"plan is {self.height}x{self.width}, data is {f.shape}")
        return replace(self, f_hat=f)


def make_plan(height: int, width: int, lam: float, c: float, f=None, workers: int = 1) -> SolverPlan:
    """solver.py:78-106 validation; device tables are built on first use."""
    if height < 1 or width < 1:
        raise ValueError(f"invalid plan size {height}x{width}")
    if not (lam > 0.0 and np.isfinite(lam)):
        raise ValueError(f"lam must be finite and positive, got {lam}")
    if not (c > 0.0 and np.isfinite(c)):
        raise ValueError(f"c must be finite and positive, got {c}")
    if workers < 1:
        raise ValueError(f"workers must be >= 1, got {workers}")
    plan = SolverPlan(int(height), int(width), float(lam), float(c), None, int(workers))
    if f is not None:
        plan = plan.with_data(f)
    return plan


def solve_ls(plan: SolverPlan, f, mu_x, mu_y, *, precision=None):
    """u = argmin of the quadratic bound energy (solver.py:109-134), on the GPU.

    numpy inputs return a float64 numpy array (C-contiguous, like the
    reference); CUDA tensors [H, W] or [B, H, W] return a CUDA tensor.
    """
    import torch

    shape = (plan.height, plan.width)
    is_t = isinstance(f, torch.Tensor)
    arrs = []
    for name, a in (("f", f), ("mu_x", mu_x), ("mu_y", mu_y)):
        shp = tuple(a.shape[-2:]) if is_t else np.shape(a)
        if shp != shape:
            raise ValueError(f"{name} has shape {tuple(np.shape(a))}, plan expects {shape}")
        arrs.append(a)
    # solve_ls takes (lam, c) from the plan; the penalty slot is unused.
    cp = to_c_params(Welsch(1.0), plan.lam, plan.c, 1)
    if is_t:
        t = [a if a.dim() == 3 else a.unsqueeze(0) for a in arrs]
        u = rt.solve_device(*t, cp)
        return u if f.dim() == 3 else u[0]
    dev = [rt.to_device_planes([np.asarray(a, dtype=np.float64)], precision) for a in arrs]
    u = rt.solve_device(*dev, cp)
    return rt.to_host_f64(u)[0]
