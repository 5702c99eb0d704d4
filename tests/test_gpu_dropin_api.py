"""The rest of the reference's public API on the GPU path (needs a B200).

grad_x / grad_y / adjoint_accumulate / aux_update / energy are exported by
the reference (pkg/src/ilsmooth/__init__.py:44-61) and run here as the
standalone field kernels (csrc/ils_elem.cuh); SolverPlan.denom / .f_hat
are the reference's arrays (solver.py:52-106), computed with the
hand-written transforms.  Goldens come from the real reference
(tests/golden/make_golden.py).  Also: the solve_ls staging and argument
contracts, the reference-side monkeypatch recipe of INTEGRATION.md, and the
misaligned-buffer checks of the C ABI.
"""

import ctypes as C
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs CUDA")]

import paper_2003_07504_b200 as ils  # noqa: E402
from paper_2003_07504_b200 import _lib, _runtime as rt  # noqa: E402

GOLD = os.path.join(os.path.dirname(__file__), "golden")
NAMES = ("fld_a", "fld_b", "fld_c")


@pytest.fixture(scope="module")
def g():
    return np.load(os.path.join(GOLD, "golden.npz"))


def test_gradients_and_adjoint_bit_exact(g):
    for name in NAMES:
        u, mx, my = g[name + "_u"], g[name + "_mx"], g[name + "_my"]
        gx, gy = ils.grad_x(u), ils.grad_y(u)
        assert gx.dtype == np.float64 and np.array_equal(gx, g[name + "_gx"]), name
        assert np.array_equal(gy, g[name + "_gy"]), name
        assert np.array_equal(ils.adjoint_accumulate(mx, my), g[name + "_adj"]), name
    with pytest.raises(ValueError, match="field shapes differ"):
        ils.adjoint_accumulate(np.zeros((3, 4)), np.zeros((4, 3)))


def test_aux_update_and_energy_match_goldens(g):
    ch, we = ils.Charbonnier(0.8, 1e-4), ils.Welsch(10 / 255)
    for name in NAMES:
        a = ils.aux_update(ch, ch.min_curvature, g[name + "_gx"])
        ref = g[name + "_aux_ch"]
        assert np.max(np.abs(a - ref)) <= 1e-13 * max(1.0, np.max(np.abs(ref))), name
        b = ils.aux_update(we, 3.0, g[name + "_gy"])
        assert np.max(np.abs(b - g[name + "_aux_we"])) <= 1e-14, name
        u, f = g[name + "_u"], g[name + "_f"]
        assert ils.energy(u, f, ch, 1.0) == pytest.approx(g[name + "_en"][0], rel=1e-12)
        assert ils.energy(u, f, we, 30.0) == pytest.approx(g[name + "_en"][1], rel=1e-12)
    with pytest.raises(ValueError, match="below the minimum"):
        ils.aux_update(ch, 1.0, np.zeros(3))
    with pytest.raises(ValueError, match="shapes differ"):
        ils.energy(np.zeros((3, 4)), np.zeros((4, 3)), ch, 1.0)


def test_field_functions_on_tensors_keep_dtype():
    x = torch.rand((2, 33, 45), device="cuda")
    gx = ils.grad_x(x)
    assert gx.dtype == torch.float32 and gx.is_cuda
    assert torch.equal(gx, torch.roll(x, -1, dims=2) - x)
    gy = ils.grad_y(x[0])
    assert torch.equal(gy, torch.roll(x[0], -1, dims=0) - x[0])
    e = ils.energy(x, x, ils.Charbonnier(0.8, 1e-4), 1.0)
    assert e.shape == (2,)
    # u = f: data term 0, the rest is lam * sum phi(grad)
    ref = sum(float(np.sum(ils.Charbonnier(0.8, 1e-4).value(d.double().cpu().numpy())))
              for d in (torch.roll(x[0], -1, 1) - x[0], torch.roll(x[0], -1, 0) - x[0]))
    assert float(e[0]) == pytest.approx(ref, rel=1e-5)


def test_energy_matches_smooth_plane_trace():
    # the standalone energy of the traced iterates equals the fused on-device trace
    f = np.random.default_rng(4).random((48, 40))
    params = ils.SmoothParams(ils.Charbonnier(0.8, 1e-4), 1.0, iters=3)
    u, tr = ils.smooth_plane(f, params, trace=True, precision="fp64")
    assert ils.energy(f, f, params.penalty, 1.0) == pytest.approx(tr.energies[0], rel=1e-12)
    assert ils.energy(u, f, params.penalty, 1.0) == pytest.approx(tr.energies[-1], rel=1e-12)


def test_plan_denom_and_f_hat_follow_the_reference_contract(g):
    from dataclasses import replace

    for name in NAMES:
        f = g[name + "_f"]
        h, w = f.shape
        plan = ils.make_plan(h, w, 1.5, 4.0, f)
        assert plan.denom.shape == (h, w) and plan.denom.dtype == np.float64
        assert np.allclose(plan.denom, g[name + "_denom"], rtol=1e-13, atol=0)  # GPU vs libm cos ulps
        assert plan.f_hat.dtype == np.complex128
        assert np.max(np.abs(plan.f_hat - g[name + "_fhat"])) <= 1e-12 * max(1.0, np.max(np.abs(g[name + "_fhat"])))
        # hqs.py:61 rebinds f_hat with dataclasses.replace
        p2 = replace(ils.make_plan(h, w, 2.0, 1.0), f_hat=plan.f_hat)
        assert p2.f_hat is plan.f_hat and p2.lam == 2.0
    assert ils.make_plan(4, 4, 1.0, 2.0).f_hat is None


def test_solve_ls_numpy_inputs_staged_once_large_plane():
    # large planes: the three inputs share one pinned staging buffer; a reuse
    # race would put mu_x's data into f
    rng = np.random.default_rng(8)
    H, W = 1080, 1920
    f, mx, my = rng.random((H, W)), 0.1 * rng.standard_normal((H, W)), 0.1 * rng.standard_normal((H, W))
    plan = ils.make_plan(H, W, 1.0, 2.0)
    u1 = ils.solve_ls(plan, f, mx, my)
    u2 = ils.solve_ls(plan, f, np.zeros_like(mx), np.zeros_like(my))
    from oracle import ils_oracle as O

    assert np.max(np.abs(u1 - O.solve_ls(f, mx, my, 1.0, 2.0, os.cpu_count() or 1))) < 1e-10  # fp64 default
    assert np.max(np.abs(u2 - O.solve_ls(f, 0 * mx, 0 * my, 1.0, 2.0, os.cpu_count() or 1))) < 1e-10


def test_solve_ls_tensor_arguments_must_agree():
    plan = ils.make_plan(8, 8, 1.0, 2.0)
    f = torch.rand((2, 8, 8), device="cuda")
    with pytest.raises(ValueError):
        ils.solve_ls(plan, f, torch.zeros((8, 8), device="cuda"), torch.zeros((2, 8, 8), device="cuda"))
    with pytest.raises(ValueError):
        ils.solve_ls(plan, f, torch.zeros((2, 8, 8), device="cuda", dtype=torch.float64), torch.zeros_like(f))
    u = ils.solve_ls(plan, f, torch.zeros_like(f), torch.zeros_like(f))
    assert u.shape == f.shape


def test_misaligned_buffers_are_rejected_or_realigned():
    # the C ABI refuses rows the TMA bulk copies cannot move ...
    params = ils.SmoothParams(ils.Charbonnier(0.8, 1e-4), 1.0)
    plan = rt.get_plan(1, 64, 1920, params.c_params(), _lib.ILS_F32, 0)
    buf = torch.rand(64 * 1920 + 8, device="cuda")
    ws = torch.empty(plan.workspace_bytes, dtype=torch.uint8, device="cuda")
    st = torch.empty(1, dtype=torch.int32, device="cuda")
    L = _lib.lib()
    s = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    rc = L.ils_smooth(plan.ptr, C.c_void_p(buf.data_ptr() + 4), C.c_void_p(buf.data_ptr()), 64 * 1920,
                      C.c_void_p(ws.data_ptr()), s, C.c_void_p(st.data_ptr()), None)
    assert rc == _lib.ILS_EINVAL and "aligned" in _lib.last_error()
    rc = L.ils_smooth(plan.ptr, C.c_void_p(buf.data_ptr()), C.c_void_p(buf.data_ptr()), 64 * 1920 + 1,
                      C.c_void_p(ws.data_ptr()), s, C.c_void_p(st.data_ptr()), None)
    assert rc == _lib.ILS_EINVAL
    # ... and the Python layer re-aligns a view at an odd storage offset
    x = buf[1:1 + 64 * 1920].view(64, 1920)
    u = ils.smooth_plane(x, params)
    ref = ils.smooth_plane(x.clone(), params)
    assert torch.equal(u, ref)


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs two GPUs")
def test_second_device_without_set_device():
    params = ils.SmoothParams(ils.Charbonnier(0.8, 1e-4), 1.0)
    x = torch.rand((3, 64, 96), device="cuda:1")
    u1 = ils.smooth_batch(x, params)
    u0 = ils.smooth_batch(x.to("cuda:0"), params)
    assert torch.equal(u1.cpu(), u0.cpu())


def _foreign_params():
    """Parameter objects of another package with the reference's fields (the
    reference's own frozen dataclasses, penalty.py:47-105, smoother.py:31-62,
    image.py:29-107), as a monkeypatched reference program passes them."""
    from dataclasses import dataclass
    from enum import Enum

    class ColorMode(Enum):
        PER_CHANNEL_RGB = "per_channel_rgb"
        LUMINANCE_ONLY = "luminance_only"

    @dataclass(frozen=True)
    class Charbonnier:
        p: float = 0.8
        eps: float = 1e-4

        @property
        def min_curvature(self):
            return self.p * self.eps ** (self.p / 2.0 - 1.0)

    @dataclass(frozen=True)
    class SmoothParams:
        penalty: object
        lam: float
        iters: int = 4
        c: float = None
        color_mode: object = ColorMode.PER_CHANNEL_RGB

        @property
        def curvature(self):
            return self.penalty.min_curvature if self.c is None else float(self.c)

    @dataclass(frozen=True)
    class MultiImage:
        channels: tuple
        space: str = "rgb"

    return Charbonnier, SmoothParams, MultiImage, ColorMode


def test_reference_monkeypatch_recipe_of_integration_md():
    # the reference's call sites patched to this
    # package, called with the reference's own parameter / image objects
    import types

    Charb, SP, MI, CM = _foreign_params()
    refmod = types.SimpleNamespace()
    for name in ("smooth_plane", "smooth_color"):
        setattr(refmod, name, getattr(ils, name))
    f = np.random.default_rng(1).random((32, 40))
    ours = ils.SmoothParams(ils.Charbonnier(0.8, 1e-4), 1.0)
    theirs = SP(Charb(0.8, 1e-4), 1.0)
    u = refmod.smooth_plane(f, theirs)
    assert u.dtype == np.float64 and u.flags["C_CONTIGUOUS"]
    assert np.array_equal(u, ils.smooth_plane(f, ours))
    rgb = np.random.default_rng(2).random((16, 14, 3))
    planes = tuple(np.ascontiguousarray(rgb[..., k]) for k in range(3))
    out = refmod.smooth_color(MI(planes, "rgb"), theirs)
    assert type(out) is MI and out.space == "rgb"
    ref = ils.smooth_color(ils.MultiImage(planes, ils.RGB), ours)
    for a, b in zip(out.channels, ref.channels):
        assert np.array_equal(a, b)
    lum = refmod.smooth_color(MI(planes, "rgb"), SP(Charb(0.8, 1e-4), 1.0, color_mode=CM.LUMINANCE_ONLY))
    lum_ref = ils.smooth_color(ils.MultiImage(planes, ils.RGB),
                               ils.SmoothParams(ils.Charbonnier(0.8, 1e-4), 1.0,
                                                color_mode=ils.ColorMode.LUMINANCE_ONLY))
    for a, b in zip(lum.channels, lum_ref.channels):
        assert np.array_equal(a, b)


def test_integration_md_ctypes_stub_runs():
    # the reference-side ctypes binding printed in INTEGRATION.md, executed as written
    import re

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    text = open(os.path.join(root, "INTEGRATION.md")).read()
    block = next(b for b in re.findall(r"```python\n(.*?)```", text, re.S) if "def smooth_plane_b200" in b)
    os.environ["ILS_B200_LIB"] = _lib.LIB_PATH
    for cand in ("/usr/local/cuda/lib64/libcudart.so", "/usr/local/cuda/lib64/libcudart.so.12"):
        if os.path.exists(cand):
            os.environ.setdefault("CUDART_LIB", cand)
    ns = {}
    exec(compile(block, "INTEGRATION.md", "exec"), ns)
    f = np.random.default_rng(3).random((48, 64))
    params = ils.SmoothParams(ils.Charbonnier(0.8, 1e-4), 1.0)
    u = ns["smooth_plane_b200"](f, params)
    assert np.array_equal(u, ils.smooth_plane(f, params))
