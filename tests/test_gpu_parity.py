"""CUDA path vs the pinned oracle and the reference goldens (needs a B200).

Tolerances (north star, BASELINE.json): fp32 max-abs <= 1e-4 on [0,1]
images and PSNR >= 60 dB against the float64 reference; the fp64
instantiation is held to the reference's own fp64-tight bounds
(pkg/tests/test_solver.py:88 1e-9, test_smoother.py:138 1e-12).
"""

import csv
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs CUDA")]

import paper_2003_07504_b200 as ils  # noqa: E402
from oracle import ils_oracle as O  # noqa: E402

GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def g():
    return np.load(os.path.join(GOLD, "golden.npz"))


def _pen_from(arr):
    kind, p, eps, gamma, lam, c, iters = arr
    if int(kind) == 0:
        return ils.Charbonnier(float(p), float(eps)), O.Charbonnier(p, eps), float(lam), float(c), int(iters)
    return ils.Welsch(float(gamma)), O.Welsch(gamma), float(lam), float(c), int(iters)


# ------------------------------------------------------------ the transform itself
@pytest.mark.parametrize("shape", [(1080, 1920), (512, 512), (17, 13), (5, 7), (33, 45), (1, 6), (3, 1), (20, 14),
                                   (2160, 3840), (48, 40), (120, 34)])
@pytest.mark.parametrize("prec", ["fp32", "fp64"])
def test_rfft2_irfft2_match_numpy(shape, prec):
    rng = np.random.default_rng(1)
    x = rng.standard_normal((2,) + shape)
    dt = torch.float32 if prec == "fp32" else torch.float64
    xt = torch.from_numpy(x).to("cuda", dt)
    X = ils._runtime.rfft2_device(xt).cpu().numpy()
    ref = np.fft.rfft2(x)
    scale = np.max(np.abs(ref))
    tol = 2e-6 if prec == "fp32" else 1e-13
    assert np.max(np.abs(X - ref)) / scale < tol
    back = ils._runtime.irfft2_device(torch.from_numpy(ref).to("cuda", torch.complex64 if prec == "fp32"
                                                                else torch.complex128), shape[1]).cpu().numpy()
    assert np.max(np.abs(back - x)) < (1e-5 if prec == "fp32" else 1e-12)


# ------------------------------------------------------------ solve_ls
@pytest.mark.parametrize("prec,tol", [("fp64", 1e-9), ("fp32", 2e-6)])  # fp32 measured 4.2e-7
def test_solve_ls_matches_reference_goldens(g, prec, tol):
    worst = 0.0
    for key in g.files:
        if key.startswith("solve_") and key.endswith("_u"):
            k = key[:-2]
            lam, c = g[k + "_lamc"]
            f, mx, my = g[k + "_f"], g[k + "_mx"], g[k + "_my"]
            plan = ils.make_plan(f.shape[0], f.shape[1], lam, c, f)
            u = ils.solve_ls(plan, f, mx, my, precision=prec)
            err = np.max(np.abs(u - g[key])) / max(1.0, np.max(np.abs(g[key])))
            worst = max(worst, err)
            assert err < tol, (k, err)
    assert worst >= 0.0


def test_solve_ls_dense_oracle_fp64():
    # reference test_solver.py:78-88 on the CUDA fp64 path
    rng = np.random.default_rng(42)
    for h, w in ((4, 4), (5, 7), (16, 16), (17, 13), (1, 6), (3, 1)):
        for lam, c in ((0.1, 2.0), (1.0, 100.0), (10.0, 2.0)):
            f, mx, my = (rng.standard_normal((h, w)) for _ in range(3))
            u = ils.solve_ls(ils.make_plan(h, w, lam, c, f), f, mx, my, precision="fp64")
            assert np.max(np.abs(u - O.dense_solve(f, mx, my, lam, c))) < 1e-9


def test_solve_ls_nonfinite_raises():
    plan = ils.make_plan(4, 4, 1.0, 2.0)
    good = np.zeros((4, 4))
    bad = good.copy()
    bad[1, 1] = np.nan
    with pytest.raises(ils.NumericalError):
        ils.solve_ls(plan, bad, good, good)
    with pytest.raises(ils.NumericalError):
        ils.solve_ls(plan, good, bad, good)
    with pytest.raises(ValueError):
        ils.solve_ls(plan, np.zeros((4, 5)), good, good)


# ------------------------------------------------------------ smooth_plane
@pytest.mark.parametrize("prec", ["fp64", "fp32"])
def test_smooth_plane_matches_reference_goldens(g, prec):
    names = sorted({k[: -len("_pen")] for k in g.files if k.endswith("_pen")})
    for name in names:
        pen, _, lam, c, iters = _pen_from(g[name + "_pen"])
        params = ils.SmoothParams(pen, lam, iters=iters, c=c)
        u, tr = ils.smooth_plane(g[name + "_f"], params, trace=True, precision=prec)
        ref = g[name + "_u"]
        err = np.max(np.abs(u - ref))
        if prec == "fp64":
            assert err < 1e-9, (name, err)
            assert np.allclose(tr.energies, g[name + "_energies"], rtol=1e-9), name
        else:
            assert err <= 1e-4, (name, err)
            assert O.psnr(u, ref) >= 60.0, name
            assert np.allclose(tr.energies, g[name + "_energies"], rtol=1e-4), name


def test_c1_512_oracle_config(g):
    # 512x512 uniform rng(0), Charbonnier p=0.8, lam=1, N=4
    f = np.random.default_rng(0).random((512, 512))
    params = ils.SmoothParams(ils.Charbonnier(0.8, 1e-4), 1.0, iters=4)
    u = ils.smooth_plane(f, params)
    ref_rows, ref_cols = g["c1_rows"], g["c1_cols"]
    assert np.max(np.abs(u[[0, 1, 255, 511], :] - ref_rows)) <= 1e-4
    assert np.max(np.abs(u[:, [0, 7, 300, 511]] - ref_cols)) <= 1e-4
    assert u.sum() == pytest.approx(g["c1_sum"][0], rel=1e-6)
    uo = O.smooth_plane(f, O.Charbonnier(0.8, 1e-4), 1.0, 4)
    assert np.max(np.abs(u - uo)) <= 1e-4
    assert O.psnr(u, uo) >= 60.0


def test_c3_1080p_rgb_batched_matches_oracle():
    planes = O.bench_planes(1080, 1920, 3)
    img = ils.MultiImage(tuple(planes), ils.RGB)
    params = ils.SmoothParams(ils.Charbonnier(0.8, 1e-4), 1.0, iters=4)
    out = ils.smooth_color(img, params)
    for ch, f in zip(out.channels, planes):
        ref = O.smooth_plane(f, O.Charbonnier(0.8, 1e-4), 1.0, 4)
        assert np.max(np.abs(ch - ref)) <= 1e-4
        assert O.psnr(ch, ref) >= 60.0


def test_c2_1080p_gray_fp64_tight():
    f = O.bench_planes(1080, 1920, 1)[0]
    u = ils.smooth_plane(f, ils.SmoothParams(ils.Charbonnier(0.8, 1e-4), 1.0), precision="fp64")
    ref = O.smooth_plane(f, O.Charbonnier(0.8, 1e-4), 1.0, 4)
    assert np.max(np.abs(u - ref)) < 1e-10


def test_texture_welsch_4k_matches_oracle():
    # C5's parameters (Welsch g=10/255, lam=30, N=10, c=2) on a 4K plane
    f = O.bench_planes(2160, 3840, 1)[0]
    params = ils.SmoothParams(ils.Welsch(10 / 255), 30.0, iters=10, c=2.0)
    u = ils.smooth_plane(f, params)
    ref = O.smooth_plane(f, O.Welsch(10 / 255), 30.0, 10, c=2.0)
    assert np.max(np.abs(u - ref)) <= 1e-4
    assert O.psnr(u, ref) >= 60.0


def test_energy_trace_golden_csv():
    # pkg/demos/out/energy_trace.csv (12 significant digits), fp64 path
    with open(os.path.join(GOLD, "energy_trace_ref.csv")) as fh:
        rows = list(csv.DictReader(fh))
    params = ils.SmoothParams(ils.Charbonnier(0.8), 1.0, iters=30)
    _, tr = ils.smooth_plane(O.make_photo(), params, trace=True, precision="fp64")
    for i, row in enumerate(rows):
        assert tr.energies[i] == pytest.approx(float(row["energy"]), rel=1e-10)
        assert tr.rel_decrease(i) == pytest.approx(float(row["rel_decrease"]), abs=1e-8)
    e = np.asarray(tr.energies)
    assert np.all(e[1:] <= e[:-1] * (1 + 1e-12))  # majorize-minimize monotonicity


# ------------------------------------------------------------ smooth_color
def test_smooth_color_rgb_and_luminance_goldens(g):
    img = ils.MultiImage.from_array(g["sc_rgb_in"])
    params = ils.SmoothParams(ils.Charbonnier(0.8, 1e-4), 1.0)
    out, tr = ils.smooth_color(img, params, trace=True, precision="fp64")
    assert np.max(np.abs(out.to_array() - g["sc_rgb_out"])) < 1e-9
    assert np.allclose(tr.energies, g["sc_rgb_energies"], rtol=1e-9)
    lum = ils.SmoothParams(ils.Charbonnier(0.8, 1e-4), 1.0, color_mode=ils.ColorMode.LUMINANCE_ONLY)
    out_l = ils.smooth_color(img, lum, precision="fp64")
    assert np.max(np.abs(out_l.to_array() - g["sc_lum_out"])) < 1e-9
    out32 = ils.smooth_color(img, params)
    assert np.max(np.abs(out32.to_array() - g["sc_rgb_out"])) <= 1e-4


def test_gray_color_matches_plane_and_rejects_yuv():
    f = np.random.default_rng(5).random((18, 22))
    params = ils.SmoothParams(ils.Charbonnier(0.8, 1e-4), 1.0)
    out = ils.smooth_color(ils.MultiImage((f,), ils.GRAY), params)
    assert np.array_equal(out.channels[0], ils.smooth_plane(f, params))
    with pytest.raises(ValueError):
        ils.smooth_color(ils.MultiImage.from_array(np.zeros((4, 4, 3)), ils.YUV), params)


# ------------------------------------------------------------ contracts
def test_fixpoints_and_determinism():
    f = np.full((20, 20), 0.42)
    params = ils.SmoothParams(ils.Charbonnier(0.8, 1e-4), 1.0)
    u = ils.smooth_plane(f, params, precision="fp64")
    assert np.max(np.abs(u - f)) < 1e-12  # test_smoother.py:134-140
    rng = np.random.default_rng(3)
    x = torch.from_numpy(rng.random((3, 1080, 1920))).to("cuda", torch.float32)
    a = ils.smooth_batch(x, params)
    b = ils.smooth_batch(x, params)
    assert torch.equal(a, b)  # bit-identical reruns (test_solver.py:172-180)
    # placement invariance: a plane smoothed alone equals it inside a batch
    c = ils.smooth_batch(x[1:2].clone(), params)
    assert torch.equal(c[0], a[1])


def test_errors_map_to_reference_exceptions():
    params = ils.SmoothParams(ils.Charbonnier(0.8, 1e-4), 1.0)
    bad = np.zeros((8, 8))
    bad[2, 2] = np.inf
    with pytest.raises(ValueError):
        ils.smooth_plane(bad, params)
    t = torch.zeros((8, 8), device="cuda")
    t[3, 3] = float("nan")
    with pytest.raises(ValueError):
        ils.smooth_plane(t, params)
    # a finite input whose iterate overflows -> NumericalError naming iteration 1
    huge = np.full((8, 8), 1e30)
    huge[::2, ::2] = -1e30
    with pytest.raises(ils.NumericalError, match="iteration"):
        ils.smooth_plane(huge, ils.SmoothParams(ils.Charbonnier(0.8, 1e-4), 1e30), precision="fp32")
    with pytest.raises(ValueError):
        ils.smooth_plane(np.zeros((8, 8)), params, plan=ils.make_plan(8, 8, 2.0, params.curvature))
    with pytest.raises(ValueError):
        ils.smooth_plane(np.zeros((8, 8)), params, plan=ils.make_plan(8, 9, 1.0, params.curvature))


def test_torch_zero_copy_path_matches_numpy_path():
    f = np.random.default_rng(9).random((64, 80))
    params = ils.SmoothParams(ils.Welsch(0.1), 2.0, iters=5)
    u_np = ils.smooth_plane(f, params)
    u_t = ils.smooth_plane(torch.from_numpy(f).to("cuda", torch.float32), params)
    assert np.array_equal(u_np, u_t.double().cpu().numpy())


@pytest.mark.parametrize("iters", [4, 3])
def test_launch_pass_sequence_equals_smooth(iters):
    # the per-pass entry point (roofline timing, bench.py) replays the exact ils_smooth dataflow
    import ctypes as C

    from paper_2003_07504_b200 import _lib, _runtime as rt

    params = ils.SmoothParams(ils.Charbonnier(0.8, 1e-4), 1.0, iters=iters)
    f = torch.rand((3, 270, 480), device="cuda", generator=torch.Generator("cuda").manual_seed(3))
    ref = ils.smooth_batch(f, params)
    plan = rt.get_plan(3, 270, 480, params.c_params(), _lib.ILS_F32, 0)
    ws = torch.empty(plan.workspace_bytes, dtype=torch.uint8, device="cuda")
    st = torch.full((1,), _lib.STATUS_CLEAN, dtype=torch.int32, device="cuda")
    u = torch.empty_like(f)
    order = [0, 1]
    for n in range(1, iters):
        cur = 0 if n % 2 else 4
        order += [2 | cur, 1 | (cur ^ 4)]
    order += [3 | (0 if iters % 2 else 4)]
    L = _lib.lib()
    s = torch.cuda.current_stream().cuda_stream
    for p in order:
        _lib.check(L.ils_launch_pass(plan.ptr, p, C.c_void_p(f.data_ptr()), C.c_void_p(u.data_ptr()), 270 * 480,
                                     C.c_void_p(ws.data_ptr()), C.c_void_p(s), C.c_void_p(st.data_ptr())),
                   "ils_launch_pass")
    torch.cuda.synchronize()
    assert torch.equal(u, ref)
    with pytest.raises(ValueError):
        _lib.check(L.ils_launch_pass(plan.ptr, 4, None, None, 0, C.c_void_p(ws.data_ptr()), C.c_void_p(s),
                                     C.c_void_p(st.data_ptr())), "ils_launch_pass")


# ------------------------------------------------------------ C5 slab decomposition (emulated ranks)
@pytest.mark.parametrize("H,W,P", [(1080, 1920, 2), (1080, 1920, 3), (256, 320, 4), (90, 128, 8)])
def test_slab_decomposition_bitwise_equals_single_gpu(H, W, P):
    from paper_2003_07504_b200.dist import EmulatedSlab

    params = ils.SmoothParams(ils.Charbonnier(0.8, 1e-4), 1.0, iters=4)
    f = torch.from_numpy(np.random.default_rng(11).random((H, W))).to("cuda", torch.float32)
    one = ils.smooth_batch(f[None], params)[0]
    em = EmulatedSlab(H, W, params, P)
    u = em.smooth(f)
    assert torch.equal(u, one)  # bitwise: every line is transformed by the same code wherever it lives


def test_c5_8k_texture_slab_and_wide_rows():
    # C5: 7680x4320, Welsch g=10/255, lam=30, N=10, c=2 (texture parameters, no pre-blur)
    from paper_2003_07504_b200.dist import EmulatedSlab

    params = ils.SmoothParams(ils.Welsch(10 / 255), 30.0, iters=10, c=2.0)
    f = torch.from_numpy(np.random.default_rng(20240607).random((4320, 7680))).to("cuda", torch.float32)
    one = ils.smooth_batch(f[None], params)[0]
    u8 = EmulatedSlab(4320, 7680, params, 8).smooth(f)
    assert torch.equal(u8, one)
    # parity of the wide-row path vs the oracle on a band-limited crop of the same width
    fc = np.random.default_rng(3).random((120, 7680))
    uc = ils.smooth_plane(fc, params)
    ref = O.smooth_plane(fc, O.Welsch(10 / 255), 30.0, 10, c=2.0)
    assert np.max(np.abs(uc - ref)) <= 1e-4


def test_slab_pipeline_nccl_one_rank_bitwise():
    # C5 driver with the exchanges overlapped (SlabPipeline, async NCCL
    # all_to_all_single on a 1-rank group): bit-identical to the 1-GPU smooth
    import socket

    import torch.distributed as dist

    from paper_2003_07504_b200 import _lib
    from paper_2003_07504_b200 import dist as D

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    own = not dist.is_initialized()
    if own:
        dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                                device_id=torch.device("cuda", 0))
    try:
        H, W = 360, 640
        params = ils.SmoothParams(ils.Welsch(10 / 255), 30.0, iters=5, c=2.0)
        img = torch.from_numpy(np.random.default_rng(5).random((3, H, W))).to("cuda", torch.float32)
        plan, lay = D.slab_layout(H, W, params.c_params(), _lib.ILS_F32, 1, 0, device=0)
        stream = lambda: torch.cuda.current_stream().cuda_stream  # noqa: E731
        pipe = D.SlabPipeline(lay, params.iters, D.CudaSlabKernels(plan, stream), D.torch_exchange_async(),
                              lambda n: torch.zeros(n, dtype=torch.float32, device="cuda"), planes=3)
        rows = D.halo_rows(H, 0, H)
        f_ext = [img[c][rows].contiguous() for c in range(3)]
        us = [torch.empty((H, W), device="cuda") for _ in range(3)]
        status = torch.full((1,), _lib.STATUS_CLEAN, dtype=torch.int32, device="cuda")
        pipe.smooth(f_ext, us, status)
        torch.cuda.synchronize()
        assert int(status.item()) == _lib.STATUS_CLEAN
        ref = ils.smooth_batch(img, params)
        for c in range(3):
            assert torch.equal(us[c], ref[c])
        _lib.lib().ils_plan_destroy(plan)
    finally:
        if own:
            dist.destroy_process_group()


def test_concurrent_lanes_bitwise_match_single_stream():
    # the bench's two-lane pattern (one plan, two workspaces, two streams, passes
    # launched with programmatic dependent launch): every frame bit-identical
    # to smoothing it alone, over repeated runs (a race would show as a flip)
    import ctypes as C

    from paper_2003_07504_b200 import _lib, _runtime as rt

    params = ils.SmoothParams(ils.Charbonnier(0.8, 1e-4), 1.0, iters=4)
    H, W, CH, F = 1080, 1920, 3, 6
    gen = torch.Generator(device="cuda").manual_seed(3)
    f = torch.rand((F * CH, H, W), generator=gen, device="cuda")
    ref = torch.stack([ils.smooth_batch(f[k * CH:(k + 1) * CH], params) for k in range(F)]).reshape(F * CH, H, W)
    plan = rt.get_plan(CH, H, W, params.c_params(), _lib.ILS_F32, 0)
    L = _lib.lib()
    lanes = [torch.cuda.Stream(), torch.cuda.Stream()]
    wss = [torch.empty(plan.workspace_bytes, dtype=torch.uint8, device="cuda") for _ in lanes]
    sts = [torch.empty(1, dtype=torch.int32, device="cuda") for _ in lanes]
    for _ in range(3):
        u = torch.empty_like(f)
        torch.cuda.synchronize()
        for k in range(F):
            ln = k % 2
            off = k * CH * H * W * 4
            _lib.check(L.ils_smooth(plan.ptr, C.c_void_p(f.data_ptr() + off), C.c_void_p(u.data_ptr() + off), H * W,
                                    C.c_void_p(wss[ln].data_ptr()), C.c_void_p(lanes[ln].cuda_stream),
                                    C.c_void_p(sts[ln].data_ptr()), None), "ils_smooth")
        torch.cuda.synchronize()
        for st in sts:
            assert int(st.item()) == _lib.STATUS_CLEAN
        assert torch.equal(u, ref)
