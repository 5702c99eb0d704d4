"""C5's 4320-point columns against the oracle and numpy (needs a B200).

The column half of every ILS iteration at 8K height runs the two-stage
register-resident solve k_col2<72, 60> (csrc/ils_col2.cuh; the reference's
column FFT -> / denom -> inverse, pkg/src/ilsmooth/solver.py:127-130), and
the standalone transforms run the Stockham k_col spec 4320 = 24*18*10.
These tests compare both with the float64 oracle / numpy.fft at H = 4320,
including one full 7680x4320 plane of the C5 configuration (Welsch
gamma = 10/255, lam = 30, N = 10, c = 2: BASELINE.json configs[4]).
Tolerance (north star): max-abs <= 1e-4 and PSNR >= 60 dB on [0, 1] images.
"""

import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs CUDA")]

import paper_2003_07504_b200 as ils  # noqa: E402
from oracle import ils_oracle as O  # noqa: E402

WORKERS = os.cpu_count() or 1
C5 = dict(gamma=10 / 255, lam=30.0, iters=10, c=2.0)


def _penalties():
    return [
        (ils.SmoothParams(ils.Charbonnier(0.8, 1e-4), 1.0, iters=4), (O.Charbonnier(0.8, 1e-4), 1.0, 4, None)),
        (ils.SmoothParams(ils.Welsch(C5["gamma"]), C5["lam"], iters=C5["iters"], c=C5["c"]),
         (O.Welsch(C5["gamma"]), C5["lam"], C5["iters"], C5["c"])),
    ]


def test_plan_uses_the_staged_4320_column_kernels():
    from paper_2003_07504_b200 import _lib, _runtime as rt

    p = rt.get_plan(1, 4320, 256, ils.SmoothParams(ils.Welsch(0.1), 1.0).c_params(), _lib.ILS_F32, 0)
    assert (p.info["col2_n1"], p.info["col2_n2"]) == (72, 60) and p.info["col3_spec"] == -1


@pytest.mark.parametrize("H", [1080, 2160, 4320])
def test_three_stage_and_two_stage_column_solves_agree(H, monkeypatch):
    # k_col3 (opt-in, ILS_COL3_SPEC=-2) and k_col2 (default) on the same plane: both
    # within the north-star tolerance of the oracle, and within fp32 noise of each other
    import ctypes as C

    from paper_2003_07504_b200 import _lib

    params = ils.SmoothParams(ils.Welsch(C5["gamma"]), C5["lam"], iters=C5["iters"], c=C5["c"])
    f = np.random.default_rng(H).random((H, 64))
    ft = torch.from_numpy(f).to("cuda", torch.float32)[None]
    L = _lib.lib()
    outs = []
    for env in ("-2", None):  # the opt-in three-stage kernel, then the default k_col2
        if env is None:
            monkeypatch.delenv("ILS_COL3_SPEC", raising=False)
        else:
            monkeypatch.setenv("ILS_COL3_SPEC", env)
        h = C.c_void_p()
        _lib.check(L.ils_plan_create(C.byref(h), 1, H, 64, C.byref(ils.penalty.params_of(params)), _lib.ILS_F32, 0))
        info = _lib.PlanInfo()
        L.ils_plan_get_info(h, C.byref(info))
        assert (info.col3_spec >= 0) == (env is not None)
        ws_sz = C.c_size_t()
        L.ils_workspace_size(h, C.byref(ws_sz))
        ws = torch.empty(ws_sz.value, dtype=torch.uint8, device="cuda")
        st = torch.empty(1, dtype=torch.int32, device="cuda")
        u = torch.empty_like(ft)
        _lib.check(L.ils_smooth(h, C.c_void_p(ft.data_ptr()), C.c_void_p(u.data_ptr()), H * 64,
                                C.c_void_p(ws.data_ptr()), C.c_void_p(torch.cuda.current_stream().cuda_stream),
                                C.c_void_p(st.data_ptr()), None))
        torch.cuda.synchronize()
        assert int(st.item()) == _lib.STATUS_CLEAN
        outs.append(u[0].double().cpu().numpy())
        L.ils_plan_destroy(h)
    ref = O.smooth_plane(f, O.Welsch(C5["gamma"]), C5["lam"], C5["iters"], c=C5["c"], workers=WORKERS)
    for u in outs:
        assert np.max(np.abs(u - ref)) <= 1e-4
    assert np.max(np.abs(outs[0] - outs[1])) <= 2e-5


@pytest.mark.parametrize("W", [64, 256])
@pytest.mark.parametrize("which", [0, 1])
def test_tall_planes_match_oracle(W, which):
    params, (pen, lam, iters, c) = _penalties()[which]
    f = np.random.default_rng(100 + W).random((4320, W))
    u = ils.smooth_plane(f, params)
    ref = O.smooth_plane(f, pen, lam, iters, c=c, workers=WORKERS)
    assert np.max(np.abs(u - ref)) <= 1e-4
    assert O.psnr(u, ref) >= 60.0


def test_tall_rgb_batch_matches_oracle():
    # three 4320-row planes in one launch sequence (channels batched)
    params, (pen, lam, iters, c) = _penalties()[1]
    planes = [np.random.default_rng(7 + k).random((4320, 128)) for k in range(3)]
    out = ils.smooth_color(ils.MultiImage(tuple(planes), ils.RGB), params)
    for ch, f in zip(out.channels, planes):
        ref = O.smooth_plane(f, pen, lam, iters, c=c, workers=WORKERS)
        assert np.max(np.abs(ch - ref)) <= 1e-4


def test_rfft2_4320_rows_matches_numpy():
    x = np.random.default_rng(2).standard_normal((2, 4320, 512))
    X = ils._runtime.rfft2_device(torch.from_numpy(x).to("cuda", torch.float32)).cpu().numpy()
    ref = np.fft.rfft2(x)
    assert np.max(np.abs(X - ref)) / np.max(np.abs(ref)) < 2e-6
    back = ils._runtime.irfft2_device(torch.from_numpy(ref).to("cuda", torch.complex64), 512).cpu().numpy()
    assert np.max(np.abs(back - x)) < 1e-5


def test_solve_ls_4320_column_solve_matches_oracle():
    # one solve_ls at H = 4320 exercises exactly the column solve k_col2<72,60> once
    rng = np.random.default_rng(9)
    f, mx, my = rng.random((4320, 96)), 0.1 * rng.standard_normal((4320, 96)), 0.1 * rng.standard_normal((4320, 96))
    plan = ils.make_plan(4320, 96, 30.0, 2.0)
    u = ils.solve_ls(plan, f, mx, my, precision="fp32")  # k_col2 is the fp32 column solve
    ref = O.solve_ls(f, mx, my, 30.0, 2.0, WORKERS)
    assert np.max(np.abs(u - ref)) <= 1e-4


def test_c5_full_8k_plane_matches_oracle():
    # BASELINE.json configs[4]: one 7680x4320 plane, C5 parameters, against the f64 oracle
    f = O.bench_planes(4320, 7680, 1)[0]
    params = ils.SmoothParams(ils.Welsch(C5["gamma"]), C5["lam"], iters=C5["iters"], c=C5["c"])
    u = ils.smooth_plane(f, params)
    ref = O.smooth_plane(f, O.Welsch(C5["gamma"]), C5["lam"], C5["iters"], c=C5["c"], workers=WORKERS)
    err = float(np.max(np.abs(u - ref)))
    assert err <= 1e-4, err
    assert O.psnr(u, ref) >= 60.0
