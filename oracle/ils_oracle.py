"""CPU oracle for the ILS smoothing hot path -- TEST INFRASTRUCTURE ONLY.

This module is a numpy/scipy restatement of the reference's algorithm
(ilsmooth, /root/reference/pkg/src/ilsmooth) for the one path this repo
accelerates: smooth_plane / smooth_color with the ILS loop
(Algorithm 1).  It exists to CHECK the CUDA product:

  * only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
    --impl reference leg may import it;
  * the product package (paper_2003_07504_b200) never imports it and has
    no CPU fallback -- it raises if the CUDA library is missing.

Parity is pinned (not just asserted): tests/test_oracle_golden.py checks
this file against golden vectors produced by importing the real reference
(tests/golden/make_golden.py, committed together with its outputs) and
against the reference's own frozen values and its committed 30-iteration
energy trace (pkg/demos/out/energy_trace.csv).

Every function cites the reference file:line it restates.  The FFT goes
through scipy.fft exactly as the reference does (solver.py:24-30), so the
restatement is bitwise-faithful on the same SciPy build.
"""

from __future__ import annotations

import numpy as np
import scipy.fft as _sfft

DEFAULT_EPS = 1e-4  # penalty.py:40
_CURVATURE_SLACK = 1e-12  # penalty.py:44


# ---------------------------------------------------------------- penalties
class Charbonnier:
    """penalty.py:47-75: (x^2+eps)^(p/2)."""

    def __init__(self, p=0.8, eps=DEFAULT_EPS):
        if not (0.0 < p <= 1.0):  # penalty.py:54-56
            raise ValueError("p must be in (0,1]")
        if not (eps > 0.0):  # penalty.py:57-58
            raise ValueError(f"eps must be positive, got {eps}")
        self.p, self.eps = float(p), float(eps)

    def value(self, x):  # penalty.py:60-62
        x = np.asarray(x, dtype=np.float64)
        return (x * x + self.eps) ** (self.p / 2.0)

    def derivative(self, x):  # penalty.py:64-66
        x = np.asarray(x, dtype=np.float64)
        return self.p * x * (x * x + self.eps) ** (self.p / 2.0 - 1.0)

    def edge_stop(self, x):  # penalty.py:68-70
        x = np.asarray(x, dtype=np.float64)
        return (self.p / 2.0) * (x * x + self.eps) ** (self.p / 2.0 - 1.0)

    @property
    def min_curvature(self):  # penalty.py:72-75
        return self.p * self.eps ** (self.p / 2.0 - 1.0)


class Welsch:
    """penalty.py:78-105: 2 g^2 (1 - exp(-x^2 / 2g^2))."""

    def __init__(self, gamma):
        if not (gamma > 0.0):  # penalty.py:84-86
            raise ValueError(f"gamma must be positive, got {gamma}")
        self.gamma = float(gamma)

    def value(self, x):  # penalty.py:88-91
        x = np.asarray(x, dtype=np.float64)
        g2 = self.gamma * self.gamma
        return 2.0 * g2 * (1.0 - np.exp(-x * x / (2.0 * g2)))

    def derivative(self, x):  # penalty.py:93-96
        x = np.asarray(x, dtype=np.float64)
        g2 = self.gamma * self.gamma
        return 2.0 * x * np.exp(-x * x / (2.0 * g2))

    def edge_stop(self, x):  # penalty.py:98-101
        x = np.asarray(x, dtype=np.float64)
        g2 = self.gamma * self.gamma
        return np.exp(-x * x / (2.0 * g2))

    @property
    def min_curvature(self):  # penalty.py:103-105
        return 2.0


def check_curvature(spec, c):
    """penalty.py:108-114."""
    c0 = spec.min_curvature
    if not np.isfinite(c) or c < c0 * (1.0 - _CURVATURE_SLACK):
        raise ValueError(f"curvature c={c} is below the minimum {c0}")


def aux_update(spec, c, x):
    """penalty.py:117-126: mu = c*x - phi'(x)."""
    check_curvature(spec, c)
    x = np.asarray(x, dtype=np.float64)
    return c * x - spec.derivative(x)


# ---------------------------------------------------------------- operators
def grad_x(u):
    """solver.py:33-35: periodic forward difference along axis 1."""
    return np.roll(u, -1, axis=1) - u


def grad_y(u):
    """solver.py:38-40: periodic forward difference along axis 0."""
    return np.roll(u, -1, axis=0) - u


def adjoint_accumulate(mu_x, mu_y):
    """solver.py:43-49: Dx^T mu_x + Dy^T mu_y (periodic)."""
    if mu_x.shape != mu_y.shape:
        raise ValueError(f"field shapes differ: {mu_x.shape} vs {mu_y.shape}")
    return np.roll(mu_x, 1, axis=1) - mu_x + np.roll(mu_y, 1, axis=0) - mu_y


def denominator(height, width, lam, c):
    """solver.py:100-102: 1 + (c lam / 2)(wy + wx), w = 2 - 2cos(2 pi k / n)."""
    wx = 2.0 - 2.0 * np.cos(2.0 * np.pi * np.arange(width) / width)
    wy = 2.0 - 2.0 * np.cos(2.0 * np.pi * np.arange(height) / height)
    return 1.0 + (c * lam / 2.0) * (wy[:, None] + wx[None, :])


def solve_ls(f, mu_x, mu_y, lam, c, workers=1, f_hat=None, denom=None):
    """solver.py:109-134: u = ifft2((fft2(f) + lam/2 fft2(D^T mu)) / denom).real."""
    h, w = f.shape
    if denom is None:
        denom = denominator(h, w, lam, c)
    if f_hat is None:
        f_hat = _sfft.fft2(f, workers=workers)
    rhs_hat = f_hat + (lam / 2.0) * _sfft.fft2(adjoint_accumulate(mu_x, mu_y), workers=workers)
    u = _sfft.ifft2(rhs_hat / denom, workers=workers)
    return np.ascontiguousarray(u.real)


def dense_solve(f, mu_x, mu_y, lam, c):
    """solver.py:152-179 restated with dense numpy matrices (<= 4096 px)."""
    h, w = f.shape
    n = h * w
    if n > 4096:
        raise ValueError("dense oracle refuses > 4096 pixels")

    def cyc(m):
        d = -np.eye(m)
        d[np.arange(m), (np.arange(m) + 1) % m] += 1.0
        return d

    dx = np.kron(np.eye(h), cyc(w))
    dy = np.kron(cyc(h), np.eye(w))
    a = np.eye(n) + (c * lam / 2.0) * (dx.T @ dx + dy.T @ dy)
    rhs = f.ravel() + (lam / 2.0) * (dx.T @ mu_x.ravel() + dy.T @ mu_y.ravel())
    return np.linalg.solve(a, rhs).reshape(h, w)


# ---------------------------------------------------------------- smoother
def energy(u, f, spec, lam):
    """smoother.py:93-101."""
    d = u - f
    return float(
        np.sum(d * d)
        + lam * (np.sum(spec.value(grad_x(u))) + np.sum(spec.value(grad_y(u))))
    )


def smooth_plane(f, spec, lam, iters=4, c=None, trace=False, workers=1):
    """smoother.py:132-172 (plan built per call, solver.py:78-106)."""
    f = np.asarray(f, dtype=np.float64)
    c = spec.min_curvature if c is None else float(c)
    h, w = f.shape
    denom = denominator(h, w, lam, c)
    f_hat = _sfft.fft2(f, workers=workers)  # SolverPlan.with_data, solver.py:69-75
    u = f
    energies = [energy(u, f, spec, lam)] if trace else None
    for n in range(iters):  # smoother.py:162-169
        mx = aux_update(spec, c, grad_x(u))
        my = aux_update(spec, c, grad_y(u))
        u = solve_ls(f, mx, my, lam, c, workers, f_hat=f_hat, denom=denom)
        if not np.all(np.isfinite(u)):
            raise ArithmeticError(f"non-finite iterate at iteration {n + 1}")
        if trace:
            energies.append(energy(u, f, spec, lam))
    return (u, energies) if trace else u


# ---------------------------------------------------------------- 8-bit I/O
def quantize(plane):
    """formats.py:25-27: floor(clip01(v) * 255 + 0.5) as uint8 (image.clip01 = np.clip(v, 0, 1))."""
    return np.floor(np.clip(plane, 0.0, 1.0) * 255.0 + 0.5).astype(np.uint8)


def smooth_u8(arr, spec, lam, iters=4, c=None, workers=1):
    """8-bit image [H, W] or [H, W, C] -> the reference's PNG round trip:
    arr / 255 (formats.py:43) -> smooth per channel -> quantize (formats.py:54-59)."""
    f = np.asarray(arr, dtype=np.float64) / 255.0
    if f.ndim == 2:
        return quantize(smooth_plane(f, spec, lam, iters, c, workers=workers))
    return np.stack([quantize(smooth_plane(f[..., k], spec, lam, iters, c, workers=workers))
                     for k in range(f.shape[-1])], axis=-1)


# ---------------------------------------------------------------- applications
def clip01(a):
    """image.py:48-50."""
    return np.clip(a, 0.0, 1.0)


def detail_enhance(planes, spec, lam, k, iters=4, c=None):
    """applications.py:80-93 (per channel)."""
    if k == 1.0:
        return [np.asarray(p) for p in planes]
    out = []
    for f in planes:
        u = smooth_plane(f, spec, lam, iters, c)
        out.append(clip01(u + k * (f - u)))
    return out


def gaussian_blur(plane, sigma):
    """applications.py:210-222."""
    from scipy.ndimage import convolve1d

    plane = np.asarray(plane, dtype=np.float64)
    if sigma == 0.0:
        return np.array(plane)
    radius = int(np.ceil(3.0 * sigma))
    x = np.arange(-radius, radius + 1, dtype=np.float64)
    kernel = np.exp(-(x * x) / (2.0 * sigma * sigma))
    kernel /= kernel.sum()
    out = convolve1d(plane, kernel, axis=0, mode="nearest")
    return convolve1d(out, kernel, axis=1, mode="nearest")


def clipart_clean(planes, gamma, lam):
    """applications.py:186-197."""
    return [clip01(smooth_plane(f, Welsch(gamma), lam, 10, 2.0)) for f in planes]


def texture_smooth(planes, gamma, lam, sigma_pre=1.0):
    """applications.py:200-207 (c defaults to Welsch's c0 = 2)."""
    return [clip01(smooth_plane(gaussian_blur(f, sigma_pre), Welsch(gamma), lam, 15)) for f in planes]


def _tonemap_finish(lum, rgb, log_lum_out, saturation):
    lum_out = 10.0 ** log_lum_out  # applications.py:121-129
    return [clip01((ch / lum) ** saturation * lum_out) for ch in rgb]


def _compress_base(base, target_range):
    spread = float(base.max() - base.min())  # applications.py:111-118
    if spread < 1e-9:
        raise ArithmeticError(f"degenerate base dynamic range {spread:g}")
    return (base - base.max()) * (target_range / spread)


def tonemap_single(lum, rgb, spec, lam, iters=4, c=None, target_range=2.0, saturation=0.6, log_offset=1e-6):
    """applications.py:132-150."""
    log_lum = np.log10(lum + log_offset)
    base = smooth_plane(log_lum, spec, lam, iters, c)
    out = _compress_base(base, target_range) + (log_lum - base)
    return _tonemap_finish(lum, rgb, out, saturation)


def tonemap_multi(lum, rgb, spec, lambdas, iters=4, c=None, target_range=2.0, saturation=0.6, log_offset=1e-6,
                  weights=(1.0, 1.0, 1.0)):
    """applications.py:153-183."""
    log_lum = np.log10(lum + log_offset)
    b = [smooth_plane(log_lum, spec, lm, iters, c) for lm in lambdas]
    w0, w1, w2 = weights
    out = _compress_base(b[2], target_range) + w2 * (b[1] - b[2]) + w1 * (b[0] - b[1]) + w0 * (log_lum - b[0])
    return _tonemap_finish(lum, rgb, out, saturation)


# ---------------------------------------------------------------- HQS baseline
def soft_threshold(x, alpha):
    """penalty.py:168-177."""
    x = np.asarray(x, dtype=np.float64)
    return np.where(np.abs(x) <= alpha, 0.0, x - alpha * np.sign(x))


def hqs_smooth_plane(f, lam, beta0=None, kappa=2.0, iters=4, workers=1):
    """hqs.py:50-66: beta_n = beta0 kappa^n, alpha_n = lam / (2 beta_n),
    m = soft_threshold(grad u, alpha_n), u = solve_ls(lam=2 beta_n, c=1)."""
    f = np.asarray(f, dtype=np.float64)
    h, w = f.shape
    beta = 2.0 * lam if beta0 is None else float(beta0)  # HqsParams.initial_beta, hqs.py:45-47
    f_hat = _sfft.fft2(f, workers=workers)  # hqs.py:52-53
    u = f
    for n in range(iters):
        b = beta * kappa ** n
        alpha = lam / (2.0 * b)
        mx = soft_threshold(grad_x(u), alpha)
        my = soft_threshold(grad_y(u), alpha)
        u = solve_ls(f, mx, my, 2.0 * b, 1.0, workers, f_hat=f_hat, denom=denominator(h, w, 2.0 * b, 1.0))
        if not np.all(np.isfinite(u)):
            raise ArithmeticError(f"non-finite iterate at iteration {n + 1}")
    return u


def rgb_to_yuv(r, g, b):
    """image.py:110-117 (BT.601)."""
    y = 0.299 * r + 0.587 * g + 0.114 * b
    return y, 0.492 * (b - y), 0.877 * (r - y)


def yuv_to_rgb(y, u, v):
    """image.py:120-128."""
    r = y + v / 0.877
    b = y + u / 0.492
    g = (y - 0.299 * r - 0.114 * b) / 0.587
    return r, g, b


def smooth_color(planes, spec, lam, iters=4, c=None, luminance_only=False, trace=False, workers=1):
    """smoother.py:175-217 for gray (1 plane) or rgb (3 planes) input.

    Per-channel RGB shares one plan (smoother.py:203-212); traced energies
    are summed across channels (213-216).  luminance_only smooths Y of the
    BT.601 decomposition and passes chroma through (195-202).
    """
    planes = [np.asarray(p, dtype=np.float64) for p in planes]
    if len(planes) == 3 and luminance_only:
        y, cu, cv = rgb_to_yuv(*planes)
        res = smooth_plane(y, spec, lam, iters, c, trace, workers)
        ys = res[0] if trace else res
        out = list(yuv_to_rgb(ys, cu, cv))
        return (out, res[1]) if trace else out
    if workers > 1 and len(planes) > 1:
        # smoother.py:203-212: per-channel smooths on a thread pool of <= 3
        # (numpy / scipy.fft release the GIL), each with the same `workers`
        from concurrent.futures import ThreadPoolExecutor

        with ThreadPoolExecutor(max_workers=min(3, len(planes), workers)) as pool:
            results = list(pool.map(lambda p: smooth_plane(p, spec, lam, iters, c, trace, workers), planes))
    else:
        results = [smooth_plane(p, spec, lam, iters, c, trace, workers) for p in planes]
    if trace:
        outs = [r[0] for r in results]
        summed = [float(sum(v)) for v in zip(*(r[1] for r in results))]
        return outs, summed
    return results


# ---------------------------------------------------------------- fixtures
def bench_planes(height, width, channels, seed=20240607):
    """The reference bench inputs: cli.py:270-273 (rng.random per plane)."""
    rng = np.random.default_rng(seed)
    return [rng.random((height, width)) for _ in range(channels)]


def make_photo(h=192, w=192, seed=3):
    """Restates demos/energy_trace.py:20-29 (the golden-trace input)."""
    rng = np.random.default_rng(seed)
    yy, xx = np.mgrid[0:h, 0:w] / h
    img = 0.35 + 0.25 * (xx + yy < 0.9)
    for _ in range(6):
        cy, cx, r = rng.random(3) * (0.8, 0.8, 0.15) + (0.1, 0.1, 0.04)
        img += 0.2 * np.exp(-((yy - cy) ** 2 + (xx - cx) ** 2) / r**2)
    img += 0.02 * rng.standard_normal((h, w))
    return np.clip(img, 0.0, 1.0)


def make_test_card(h=192, w=256, seed=7):
    """Restates demos/smooth_basics.py:22-31."""
    rng = np.random.default_rng(seed)
    yy, xx = np.mgrid[0:h, 0:w]
    img = np.full((h, w), 0.25)
    img[20:90, 20:110] = 0.8
    img[(yy - 130) ** 2 + (xx - 70) ** 2 <= 35**2] = 0.55
    img[30:80, 130:240] += 0.3 * (xx[30:80, 130:240] - 130) / 110
    img[110:180, 130:240] += 0.08 * np.sin(xx[110:180, 130:240] * 1.1)
    img += 0.03 * rng.standard_normal((h, w))
    return np.clip(img, 0.0, 1.0)


def psnr(a, b, peak=1.0):
    mse = float(np.mean((np.asarray(a, np.float64) - np.asarray(b, np.float64)) ** 2))
    return float("inf") if mse == 0.0 else 10.0 * np.log10(peak * peak / mse)
