"""Generate golden vectors by running the REAL reference (ilsmooth) in-process.

Run in the build container only (needs /root/reference, read-only):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Writes tests/golden/golden.npz.  The GPU box never runs this script; the
committed .npz travels with the repo.  Inputs are stored alongside the
outputs so the fixtures do not depend on numpy's RNG stream staying put.
"""

from __future__ import annotations

import os
import sys
from dataclasses import replace

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

import ilsmooth as ref  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.npz")


def main():
    g = {}
    # --- solve_ls vs the reference (test_solver.py:78-88 shapes + a few more)
    solver_shapes = [(4, 4), (5, 7), (16, 16), (17, 13), (1, 6), (3, 1), (9, 11), (20, 14), (32, 24), (12, 10)]
    rng = np.random.default_rng(42)
    for i, (h, w) in enumerate(solver_shapes):
        for j, (lam, c) in enumerate(((0.1, 2.0), (1.0, 100.0), (10.0, 2.0))):
            f = rng.standard_normal((h, w))
            mx = rng.standard_normal((h, w))
            my = rng.standard_normal((h, w))
            u = ref.solve_ls(ref.make_plan(h, w, lam, c, f), f, mx, my)
            k = f"solve_{i}_{j}"
            g[k + "_f"], g[k + "_mx"], g[k + "_my"], g[k + "_u"] = f, mx, my, u
            g[k + "_lamc"] = np.array([lam, c])

    # --- smooth_plane (Charbonnier / Welsch), smoother.py:132-172
    cases = [
        ("sp_uniform_18x22", np.random.default_rng(5).random((18, 22)), ref.Charbonnier(0.8, 1e-4), 1.0, 4, None),
        ("sp_uniform_64x80", np.random.default_rng(11).random((64, 80)), ref.Charbonnier(0.8, 1e-4), 1.0, 4, None),
        ("sp_welsch_20x20", np.random.default_rng(10).random((20, 20)), ref.Welsch(0.1), 2.0, 5, None),
        ("sp_p05_c4_48x40", np.random.default_rng(12).random((48, 40)), ref.Charbonnier(0.5, 1e-3), 3.0, 6, 4.0 * ref.Charbonnier(0.5, 1e-3).min_curvature),
        ("sp_odd_33x45", np.random.default_rng(13).random((33, 45)), ref.Charbonnier(0.8, 1e-4), 1.0, 4, None),
        ("sp_prime_17x13", np.random.default_rng(14).random((17, 13)), ref.Charbonnier(1.0, 1e-4), 0.5, 3, None),
        ("sp_card_192x256", None, ref.Charbonnier(0.8, 1e-4), 1.0, 4, None),
        ("sp_texture_welsch_60x45", np.random.default_rng(15).random((60, 45)), ref.Welsch(10 / 255), 30.0, 10, 2.0),
    ]
    for name, f, pen, lam, iters, c in cases:
        if f is None:
            import importlib.util
            spec = importlib.util.spec_from_file_location("sb", "/root/reference/pkg/demos/smooth_basics.py")
            sb = importlib.util.module_from_spec(spec)
            spec.loader.exec_module(sb)
            f = sb.make_test_card()
        params = ref.SmoothParams(pen, lam, iters=iters, c=c)
        u, tr = ref.smooth_plane(f, params, trace=True)
        g[name + "_f"] = f
        g[name + "_u"] = u
        g[name + "_energies"] = np.array(tr.energies)
        if isinstance(pen, ref.Charbonnier):
            g[name + "_pen"] = np.array([0, pen.p, pen.eps, 0.0, lam, params.curvature, iters])
        else:
            g[name + "_pen"] = np.array([1, 0.0, 0.0, pen.gamma, lam, params.curvature, iters])

    # --- smooth_color (smoother.py:175-217)
    rgb = np.random.default_rng(6).random((16, 14, 3))
    img = ref.MultiImage.from_array(rgb)
    params = ref.SmoothParams(ref.Charbonnier(0.8, 1e-4), 1.0)
    out, tr = ref.smooth_color(img, params, trace=True)
    g["sc_rgb_in"] = rgb
    g["sc_rgb_out"] = out.to_array()
    g["sc_rgb_energies"] = np.array(tr.energies)
    lum = replace(params, color_mode=ref.ColorMode.LUMINANCE_ONLY)
    out_l = ref.smooth_color(img, lum)
    g["sc_lum_out"] = out_l.to_array()

    # --- C1 oracle config: 512x512 uniform rng(0), N=4, p=0.8.
    # Stored as a checksum set, not the full plane.
    f = np.random.default_rng(0).random((512, 512))
    u = ref.smooth_plane(f, ref.SmoothParams(ref.Charbonnier(0.8, 1e-4), 1.0, iters=4))
    g["c1_sum"] = np.array([u.sum(), (u * u).sum(), u.min(), u.max()])
    g["c1_rows"] = u[[0, 1, 255, 511], :]  # four full rows for pointwise checks
    g["c1_cols"] = u[:, [0, 7, 300, 511]]

    # --- HQS penalty-splitting baseline (hqs.py:50-66; test_hqs.py cases + sizes the FFT plans care about)
    clean = np.full((32, 32), 0.25)
    clean[:, 16:] = 0.75
    noisy = np.clip(clean + 0.05 * np.random.default_rng(4).standard_normal((32, 32)), 0.0, 1.0)
    hqs_cases = [
        ("hqs_sched_20x16", np.random.default_rng(2).random((20, 16)), 0.25, None, 2.0, 4),
        ("hqs_noise_32x32", noisy, 0.25, None, 2.0, 4),
        ("hqs_beta_33x45", np.random.default_rng(21).random((33, 45)), 0.1, 0.5, 1.5, 6),
        ("hqs_prime_17x13", np.random.default_rng(22).random((17, 13)), 1.0, None, 3.0, 3),
        ("hqs_card_96x128", np.random.default_rng(23).random((96, 128)), 0.05, None, 2.0, 5),
    ]
    for name, f, lam, beta0, kappa, iters in hqs_cases:
        u = ref.hqs_smooth_plane(f, ref.HqsParams(lam, beta0=beta0, kappa=kappa, iters=iters))
        g[name + "_f"] = f
        g[name + "_u"] = u
        g[name + "_prm"] = np.array([lam, -1.0 if beta0 is None else beta0, kappa, iters])

    # --- 8-bit round trip through the reference's own codec path (formats.py read/quantize/write)
    import tempfile

    from ilsmooth import formats as F

    for name, shape, params in (
        ("u8_rgb", (24, 20, 3), ref.SmoothParams(ref.Charbonnier(0.8, 1e-4), 1.0)),
        ("u8_gray", (30, 18), ref.SmoothParams(ref.Welsch(10 / 255), 30.0, iters=10, c=2.0)),
    ):
        arr = np.random.default_rng(31).integers(0, 256, size=shape, dtype=np.uint8)
        with tempfile.TemporaryDirectory() as d:
            src, dst = os.path.join(d, "in.ppm" if len(shape) == 3 else "in.png"), os.path.join(d, "out.png")
            if len(shape) == 3:
                F.write_image(src, ref.MultiImage.from_array(arr / 255.0))
            else:
                F.write_image(src, ref.MultiImage((arr / 255.0,), ref.GRAY))
            img = F.read_image(src)
            assert np.array_equal(np.rint(img.to_array() * 255).astype(np.uint8), arr)
            F.write_image(dst, ref.smooth_color(img, params))
            from PIL import Image

            with Image.open(dst) as im:
                out = np.asarray(im).copy()
        g[name + "_in"] = arr
        g[name + "_out"] = out

    # --- applications (applications.py:80-222), small inputs through the real presets
    rng = np.random.default_rng(41)
    img = ref.MultiImage.from_array(rng.random((18, 22, 3)))
    g["app_img"] = img.to_array()
    prm = ref.SmoothParams(ref.Charbonnier(0.8, 1e-4), 1.0)
    g["app_detail3"] = ref.detail_enhance(img, prm, ref.DetailBoost(3.0)).to_array()
    g["app_detail0"] = ref.detail_enhance(img, prm, ref.DetailBoost(0.0)).to_array()
    g["app_clipart"] = ref.clipart_clean(img, 10 / 255, 20.0).to_array()
    g["app_texture"] = ref.texture_smooth(img, 10 / 255, 30.0, sigma_pre=1.0).to_array()
    g["app_blur15"] = ref.gaussian_blur(img.channels[0], 1.5)
    g["app_blur07"] = ref.gaussian_blur(img.channels[1], 0.7)
    lum = 10.0 ** rng.uniform(-2, 2, (24, 20))
    tint = np.stack([np.full(lum.shape, 0.9), np.full(lum.shape, 0.7), np.full(lum.shape, 0.5)], -1)
    rgb = ref.MultiImage.from_array(lum[..., None] * tint, ref.RGB)
    y = ref.luminance(rgb)
    g["app_hdr_rgb"] = rgb.to_array()
    tp = ref.TonemapParams(ref.SmoothParams(ref.Charbonnier(1.0, 1e-4), 2.0), target_range=1.5)
    g["app_tm_single"] = ref.tonemap_single(y, rgb, tp).to_array()
    tpm = ref.TonemapParams(ref.SmoothParams(ref.Charbonnier(1.0, 1e-4), 5.0), lambdas=(0.125, 1.0, 8.0),
                            weights=(1.2, 0.8, 1.0))
    g["app_tm_multi"] = ref.tonemap_multi(y, rgb, tpm).to_array()

    # --- the standalone field functions of the public API (solver.py:33-49,
    # penalty.py:117-126, smoother.py:93-101) and the plan's arrays (solver.py:69-75, 100-102)
    rng = np.random.default_rng(51)
    for name, shape in (("fld_a", (17, 13)), ("fld_b", (64, 80)), ("fld_c", (1, 6))):
        u, f = rng.random(shape), rng.random(shape)
        mx, my = rng.standard_normal(shape), rng.standard_normal(shape)
        g[name + "_u"], g[name + "_f"], g[name + "_mx"], g[name + "_my"] = u, f, mx, my
        g[name + "_gx"], g[name + "_gy"] = ref.grad_x(u), ref.grad_y(u)
        g[name + "_adj"] = ref.adjoint_accumulate(mx, my)
        ch, we = ref.Charbonnier(0.8, 1e-4), ref.Welsch(10 / 255)
        g[name + "_aux_ch"] = ref.aux_update(ch, ch.min_curvature, g[name + "_gx"])
        g[name + "_aux_we"] = ref.aux_update(we, 3.0, g[name + "_gy"])
        g[name + "_en"] = np.array([ref.energy(u, f, ch, 1.0), ref.energy(u, f, we, 30.0)])
        plan = ref.make_plan(shape[0], shape[1], 1.5, 4.0, f)
        g[name + "_denom"], g[name + "_fhat"] = plan.denom, plan.f_hat

    np.savez_compressed(OUT, **g)
    print(f"wrote {OUT} ({os.path.getsize(OUT)} bytes, {len(g)} arrays)")


if __name__ == "__main__":
    main()
