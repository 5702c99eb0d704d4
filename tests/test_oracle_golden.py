"""Pin the CPU oracle to the reference before trusting it (CPU-only).

Golden sources:
  * tests/golden/golden.npz -- produced by tests/golden/make_golden.py, which
    imports the real reference (ilsmooth) and runs it on stored inputs;
  * tests/golden/energy_trace_ref.csv -- the reference's committed 30-iteration
    trace (pkg/demos/out/energy_trace.csv:1-32);
  * frozen values from pkg/tests/test_penalty.py:17-45.
"""

import csv
import os

import numpy as np
import pytest

from oracle import ils_oracle as O

GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def g():
    return np.load(os.path.join(GOLD, "golden.npz"))


def _pen(arr):
    kind, p, eps, gamma, lam, c, iters = arr
    spec = O.Charbonnier(p, eps) if int(kind) == 0 else O.Welsch(gamma)
    return spec, lam, c, int(iters)


def test_frozen_penalty_values():
    # pkg/tests/test_penalty.py:17-34
    assert float(O.Charbonnier(1.0, 1e-4).derivative(0.1)) == pytest.approx(0.995037190209989, abs=1e-14)
    assert float(O.Charbonnier(1.0, 1e-4).edge_stop(1.0)) == pytest.approx(0.4999750018748438, abs=1e-14)
    assert float(O.Charbonnier(0.8, 1e-4).value(0.0)) == pytest.approx(0.025118864315095798, abs=1e-14)
    assert float(O.Welsch(0.5).value(0.5)) == pytest.approx(0.1967346701436833, abs=1e-14)
    assert float(O.Welsch(0.5).derivative(0.5)) == pytest.approx(0.6065306597126334, abs=1e-14)
    assert float(O.Welsch(10 / 255).edge_stop(0.1)) == pytest.approx(0.038725770351664364, abs=1e-14)


def test_frozen_min_curvatures():
    # pkg/tests/test_penalty.py:37-45
    assert O.Charbonnier(0.8, 1e-4).min_curvature == pytest.approx(200.95091452076636, rel=1e-14)
    assert O.Charbonnier(1.0, 1e-4).min_curvature == pytest.approx(100.0, rel=1e-14)
    assert O.Charbonnier(0.2, 1e-4).min_curvature == pytest.approx(796.2143411069947, rel=1e-14)
    assert O.Welsch(0.3).min_curvature == 2.0


def test_solve_matches_reference_goldens(g):
    n = 0
    for key in g.files:
        if key.startswith("solve_") and key.endswith("_u"):
            k = key[:-2]
            lam, c = g[k + "_lamc"]
            u = O.solve_ls(g[k + "_f"], g[k + "_mx"], g[k + "_my"], lam, c)
            assert np.max(np.abs(u - g[key])) < 1e-12, k
            n += 1
    assert n == 30


def test_dense_solve_agrees_with_spectral(g):
    # pkg/tests/test_solver.py:78-88 restated on the oracle
    for key in ("solve_0_0", "solve_1_1", "solve_3_2", "solve_4_0", "solve_5_1"):
        lam, c = g[key + "_lamc"]
        ud = O.dense_solve(g[key + "_f"], g[key + "_mx"], g[key + "_my"], lam, c)
        assert np.max(np.abs(ud - g[key + "_u"])) < 1e-9


def test_smooth_plane_matches_reference_goldens(g):
    names = sorted({k[: -len("_pen")] for k in g.files if k.endswith("_pen")})
    assert len(names) == 8
    for name in names:
        spec, lam, c, iters = _pen(g[name + "_pen"])
        u, en = O.smooth_plane(g[name + "_f"], spec, lam, iters, c, trace=True)
        assert np.max(np.abs(u - g[name + "_u"])) < 1e-12, name
        assert np.allclose(en, g[name + "_energies"], rtol=1e-12), name


def test_smooth_color_matches_reference_goldens(g):
    rgb = g["sc_rgb_in"]
    planes = [rgb[:, :, i] for i in range(3)]
    out, en = O.smooth_color(planes, O.Charbonnier(0.8, 1e-4), 1.0, trace=True)
    assert np.max(np.abs(np.stack(out, -1) - g["sc_rgb_out"])) < 1e-12
    assert np.allclose(en, g["sc_rgb_energies"], rtol=1e-12)
    out_l = O.smooth_color(planes, O.Charbonnier(0.8, 1e-4), 1.0, luminance_only=True)
    assert np.max(np.abs(np.stack(out_l, -1) - g["sc_lum_out"])) < 1e-12


def test_c1_config_checksums(g):
    # 512x512 uniform rng(0), Charbonnier p=0.8, lam=1, N=4
    f = np.random.default_rng(0).random((512, 512))
    u = O.smooth_plane(f, O.Charbonnier(0.8, 1e-4), 1.0, 4)
    s = g["c1_sum"]
    assert u.sum() == pytest.approx(s[0], rel=1e-12)
    assert (u * u).sum() == pytest.approx(s[1], rel=1e-12)
    assert np.max(np.abs(u[[0, 1, 255, 511], :] - g["c1_rows"])) < 1e-12
    assert np.max(np.abs(u[:, [0, 7, 300, 511]] - g["c1_cols"])) < 1e-12


def test_golden_energy_trace_csv():
    # pkg/demos/energy_trace.py:20-44 -> pkg/demos/out/energy_trace.csv
    with open(os.path.join(GOLD, "energy_trace_ref.csv")) as fh:
        rows = list(csv.DictReader(fh))
    assert len(rows) == 31
    _, en = O.smooth_plane(O.make_photo(), O.Charbonnier(0.8), 1.0, 30, trace=True)
    e0, elast = en[0], en[-1]
    for i, row in enumerate(rows):
        assert f"{en[i]:.12g}" == row["energy"], i
        rel = 1.0 if e0 == elast else (e0 - en[i]) / (e0 - elast)
        assert f"{rel:.12g}" == row["rel_decrease"], i


def _hqs_cases(g):
    return sorted({k[: -len("_prm")] for k in g.files if k.startswith("hqs_") and k.endswith("_prm")})


def test_hqs_matches_reference_goldens(g):
    # hqs.py:50-66 via tests/golden/make_golden.py (test_hqs.py inputs + extra sizes/schedules)
    names = _hqs_cases(g)
    assert len(names) == 5
    for name in names:
        lam, beta0, kappa, iters = g[name + "_prm"]
        u = O.hqs_smooth_plane(g[name + "_f"], lam, None if beta0 < 0 else beta0, kappa, int(iters))
        assert np.max(np.abs(u - g[name + "_u"])) < 1e-12, name


def test_hqs_field_step_is_grid_optimal():
    # pkg/tests/test_hqs.py:34-46 restated on the oracle's soft threshold
    rng = np.random.default_rng(0)
    grid = np.linspace(-3.0, 3.0, 12001)
    for _ in range(40):
        x, beta, lam = rng.uniform(-2, 2), rng.uniform(0.1, 5.0), rng.uniform(0.05, 2.0)
        m = float(O.soft_threshold(x, lam / (2 * beta)))
        assert beta * (x - m) ** 2 + lam * abs(m) <= float((beta * (x - grid) ** 2 + lam * np.abs(grid)).min()) + 1e-7


def test_u8_round_trip_matches_reference_codec_path(g):
    # formats.py:25-27,43 through the reference's own PNG/PPM writer and reader (make_golden.py)
    a = O.smooth_u8(g["u8_rgb_in"], O.Charbonnier(0.8, 1e-4), 1.0)
    assert np.array_equal(a, g["u8_rgb_out"])
    b = O.smooth_u8(g["u8_gray_in"], O.Welsch(10 / 255), 30.0, 10, 2.0)
    assert np.array_equal(b, g["u8_gray_out"])


def test_applications_match_reference_goldens(g):
    # applications.py:80-222 via tests/golden/make_golden.py
    img = g["app_img"]
    planes = [img[..., k] for k in range(3)]
    st = lambda ps: np.stack(ps, -1)  # noqa: E731
    cb = O.Charbonnier(0.8, 1e-4)
    assert np.max(np.abs(st(O.detail_enhance(planes, cb, 1.0, 3.0)) - g["app_detail3"])) < 1e-12
    assert np.max(np.abs(st(O.detail_enhance(planes, cb, 1.0, 0.0)) - g["app_detail0"])) < 1e-12
    assert np.max(np.abs(st(O.clipart_clean(planes, 10 / 255, 20.0)) - g["app_clipart"])) < 1e-12
    assert np.max(np.abs(st(O.texture_smooth(planes, 10 / 255, 30.0, 1.0)) - g["app_texture"])) < 1e-12
    assert np.array_equal(O.gaussian_blur(planes[0], 1.5), g["app_blur15"])
    assert np.array_equal(O.gaussian_blur(planes[1], 0.7), g["app_blur07"])
    rgb = g["app_hdr_rgb"]
    ch = [rgb[..., k] for k in range(3)]
    y = 0.299 * ch[0] + 0.587 * ch[1] + 0.114 * ch[2]
    c1 = O.Charbonnier(1.0, 1e-4)
    got = st(O.tonemap_single(y, ch, c1, 2.0, target_range=1.5))
    assert np.max(np.abs(got - g["app_tm_single"])) < 1e-12
    got = st(O.tonemap_multi(y, ch, c1, (0.125, 1.0, 8.0), weights=(1.2, 0.8, 1.0)))
    assert np.max(np.abs(got - g["app_tm_multi"])) < 1e-12


def test_field_functions_match_reference_goldens(g):
    # grad_x / grad_y / adjoint_accumulate / aux_update / energy (solver.py:33-49,
    # penalty.py:117-126, smoother.py:93-101) and the plan arrays (solver.py:69-75, 100-102)
    for name in ("fld_a", "fld_b", "fld_c"):
        u, f, mx, my = (g[name + k] for k in ("_u", "_f", "_mx", "_my"))
        assert np.array_equal(O.grad_x(u), g[name + "_gx"])
        assert np.array_equal(O.grad_y(u), g[name + "_gy"])
        assert np.array_equal(O.adjoint_accumulate(mx, my), g[name + "_adj"])
        ch, we = O.Charbonnier(0.8, 1e-4), O.Welsch(10 / 255)
        assert np.array_equal(O.aux_update(ch, ch.min_curvature, g[name + "_gx"]), g[name + "_aux_ch"])
        assert np.array_equal(O.aux_update(we, 3.0, g[name + "_gy"]), g[name + "_aux_we"])
        assert O.energy(u, f, ch, 1.0) == g[name + "_en"][0]
        assert O.energy(u, f, we, 30.0) == g[name + "_en"][1]
        h, w = u.shape
        assert np.array_equal(O.denominator(h, w, 1.5, 4.0), g[name + "_denom"])
        assert np.allclose(np.fft.fft2(f), g[name + "_fhat"], rtol=0, atol=1e-12)
