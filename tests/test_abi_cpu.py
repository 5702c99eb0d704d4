"""CPU-only checks of the C ABI boundary and host logic (no kernels launched)."""

import ctypes as C
import os
import re

import numpy as np
import pytest

import paper_2003_07504_b200 as ils
from paper_2003_07504_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _header_symbols():
    txt = open(os.path.join(ROOT, "include", "ils_b200.h")).read()
    return sorted(set(re.findall(r"ILS_API\s+[\w\s\*]+?\b(ils_\w+)\s*\(", txt)))


def test_library_loads_and_exports_every_header_symbol():
    L = _lib.lib()
    syms = _header_symbols()
    assert len(syms) == 38
    for s in syms:
        assert hasattr(L, s), s
    assert set(syms) == set(_lib.EXPORTS)
    assert L.ils_abi_version() == 1


def test_library_is_built_for_sm_100a():
    import subprocess

    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def _host_plan(b, h, w, params, dtype=_lib.ILS_F32):
    L = _lib.lib()
    p = C.c_void_p()
    st = L.ils_plan_create(C.byref(p), b, h, w, C.byref(params), dtype, -1)
    return st, p


@pytest.mark.parametrize("shape", [(1080, 1920), (512, 512), (17, 13), (5, 7), (2160, 3840), (1, 6), (3, 1),
                                   (33, 45), (720, 1280), (59, 118)])
@pytest.mark.parametrize("dtype", [_lib.ILS_F32, _lib.ILS_F64])
def test_host_planner_radix_products(shape, dtype):
    h, w = shape
    prm = ils.SmoothParams(ils.Charbonnier(0.8), 1.0).c_params()
    st, p = _host_plan(3, h, w, prm, dtype)
    assert st == 0, _lib.last_error()
    info = _lib.PlanInfo()
    assert _lib.lib().ils_plan_get_info(p, C.byref(info)) == 0
    d = info.as_dict()
    n_row = w // 2 if w % 2 == 0 else w
    assert int(np.prod(d["row_radix"] or [1])) == n_row
    assert int(np.prod(d["col_radix"] or [1])) == h
    assert all(r <= 61 for r in d["row_radix"] + d["col_radix"])
    assert d["row_smem"] <= 227 * 1024 and d["col_smem"] <= 227 * 1024
    assert d["spec_pitch"] >= w // 2 + 1
    assert d["launches_per_call"] == 2 * 4 + 1
    ws = C.c_size_t()
    assert _lib.lib().ils_workspace_size(p, C.byref(ws)) == 0
    assert ws.value >= 2 * 3 * h * (w // 2 + 1) * (8 if dtype == _lib.ILS_F32 else 16)
    _lib.lib().ils_plan_destroy(p)


def test_hot_sizes_use_compile_time_plans():
    prm = ils.SmoothParams(ils.Charbonnier(0.8), 1.0).c_params()
    st, p = _host_plan(3, 1080, 1920, prm)
    info = _lib.PlanInfo()
    _lib.lib().ils_plan_get_info(p, C.byref(info))
    assert info.row_spec >= 0 and info.col_spec >= 0
    _lib.lib().ils_plan_destroy(p)


@pytest.mark.parametrize("h,w,n1n2", [(1080, 1920, (30, 36)), (2160, 3840, (48, 45)), (4320, 7680, (72, 60)),
                                      (512, 512, None)])
def test_column_solve_kernel_choice(h, w, n1n2):
    # heights with a two-stage split run k_col2 (fp32); the 1080p row plan is
    # the padded 32 x 30 plan budgeted for 3 CTAs per SM (band 6)
    prm = ils.SmoothParams(ils.Charbonnier(0.8), 1.0).c_params()
    st, p = _host_plan(3, h, w, prm)
    assert st == 0
    info = _lib.PlanInfo()
    _lib.lib().ils_plan_get_info(p, C.byref(info))
    d = info.as_dict()
    if n1n2 is None:
        assert d["col2_spec"] == -1 and d["col3_spec"] == -1
    else:
        assert d["col2_spec"] >= 0 and (d["col2_n1"], d["col2_n2"]) == n1n2
        assert d["col2_n1"] * d["col2_n2"] == h
        assert d["col3_spec"] == -1  # the three-stage kernel is opt-in (ILS_COL3_SPEC)
    if (h, w) == (1080, 1920):
        assert d["row_radix"] == [32, 30] and d["row_swz"] == 3 and d["row_band"] == 6
        assert 3 * (d["row_smem"] + 1024) <= 228 * 1024
    _lib.lib().ils_plan_destroy(p)
    st, p64 = _host_plan(3, h, w, prm, _lib.ILS_F64)
    if st == 0:  # (fp64 8K rows exceed the row kernel's shared memory: no fp64 plan there)
        info = _lib.PlanInfo()
        assert _lib.lib().ils_plan_get_info(p64, C.byref(info)) == 0
        assert info.col2_spec == -1  # fp64 keeps the Stockham column kernel
        _lib.lib().ils_plan_destroy(p64)


def test_u8_ingest_newton_division_is_exact():
    # k_u8_planar's v/255: q = v*(1/255), q += fma(-q, 255, v) * (1/255) -- equal to the
    # correctly rounded fp32 v/255 for every byte (emulated with exact float64 FMAs)
    v = np.arange(256, dtype=np.float32)
    exact = (v.astype(np.float64) / 255.0).astype(np.float32)
    r = np.float32(1.0) / np.float32(255.0)
    q = (v * r).astype(np.float32)
    res = (v.astype(np.float64) - q.astype(np.float64) * 255.0).astype(np.float32)
    q2 = (res.astype(np.float64) * np.float64(r) + q.astype(np.float64)).astype(np.float32)
    assert np.array_equal(q2, exact)
    assert not np.array_equal(q, exact)  # the plain reciprocal product is not


def test_unsupported_prime_and_bad_params_map_to_valueerror():
    prm = ils.SmoothParams(ils.Charbonnier(0.8), 1.0).c_params()
    # primes > 61 plan onto the direct-DFT pass, up to one output per register
    # slot of a 256-thread group (16 fp32 / 8 fp64 per thread)
    for h, w, dt in [(1031, 64, _lib.ILS_F32), (97, 1, _lib.ILS_F32), (1919, 2 * 1009, _lib.ILS_F32),
                     (2039, 6, _lib.ILS_F64), (4093, 64, _lib.ILS_F32)]:
        st, p = _host_plan(1, h, w, prm, dt)
        assert st == 0, (h, w, dt)
        info = _lib.PlanInfo()
        assert _lib.lib().ils_plan_get_info(p, C.byref(info)) == 0
        assert max(info.col_radix) == max(q for q in range(2, h + 1) if h % q == 0 and
                                          all(q % d for d in range(2, q)))
        _lib.lib().ils_plan_destroy(p)
    for h, dt, nt in [(5000, _lib.ILS_F32, 512), (8192, _lib.ILS_F32, 512), (4100, _lib.ILS_F64, 512),
                      (1080, _lib.ILS_F32, 256)]:
        st, p = _host_plan(1, h, 64, prm, dt)  # long columns: 512-thread k_col groups
        assert st == 0, (h, dt)
        info = _lib.PlanInfo()
        assert _lib.lib().ils_plan_get_info(p, C.byref(info)) == 0
        assert info.col_threads == nt
        _lib.lib().ils_plan_destroy(p)
    st, _ = _host_plan(1, 4099, 64, prm)
    assert st == _lib.ILS_EUNSUPPORTED
    assert _host_plan(1, 2053, 64, prm, _lib.ILS_F64)[0] == _lib.ILS_EUNSUPPORTED
    with pytest.raises(ValueError, match="prime factor"):
        _lib.check(st)
    bad = _lib.Params(_lib.ILS_CHARBONNIER, 1.5, 1e-4, 0.0, 1.0, 300.0, 4)
    st, _ = _host_plan(1, 8, 8, bad)
    assert st == _lib.ILS_EINVAL
    with pytest.raises(ValueError, match=r"p must be in \(0,1\]"):
        _lib.check(st)
    low_c = _lib.Params(_lib.ILS_WELSCH, 0.0, 0.0, 0.1, 1.0, 1.0, 4)
    assert _host_plan(1, 8, 8, low_c)[0] == _lib.ILS_EINVAL
    zero_iters = _lib.Params(_lib.ILS_WELSCH, 0.0, 0.0, 0.1, 1.0, 2.0, 0)
    assert _host_plan(1, 8, 8, zero_iters)[0] == _lib.ILS_EINVAL


def test_host_only_plan_refuses_to_run():
    prm = ils.SmoothParams(ils.Charbonnier(0.8), 1.0).c_params()
    st, p = _host_plan(1, 8, 8, prm)
    buf = (C.c_char * 4096)()
    st = _lib.lib().ils_smooth(p, buf, buf, 64, buf, None, buf, None)
    assert st == _lib.ILS_EINVAL
    _lib.lib().ils_plan_destroy(p)


def test_status_mapping():
    with pytest.raises(ils.NumericalError):
        _lib.check(_lib.ILS_ENONFINITE)
    with pytest.raises(RuntimeError):
        _lib.check(_lib.ILS_ECUDA)
    _lib.check(_lib.ILS_OK)


def test_params_validation_mirrors_reference():
    # pkg/tests/test_smoother.py:42-57 and test_penalty.py:93-103
    pen = ils.Charbonnier(0.8, 1e-4)
    for kw in (dict(lam=0.0), dict(lam=-2.0), dict(lam=1.0, iters=0), dict(lam=1.0, c=pen.min_curvature / 2),
               dict(lam=1.0, color_mode="rgb")):
        with pytest.raises(ValueError):
            ils.SmoothParams(pen, **kw)
    with pytest.raises(ValueError, match=r"p must be in \(0,1\]"):
        ils.Charbonnier(1.2)
    with pytest.raises(ValueError):
        ils.Welsch(0.0)
    assert ils.SmoothParams(pen, 1.0).curvature == pen.min_curvature
    assert ils.Charbonnier(0.8, 1e-4).min_curvature == pytest.approx(200.95091452076636, rel=1e-14)
    for args in ((0, 4, 1.0, 2.0), (4, 4, -1.0, 2.0), (4, 4, 1.0, 0.0)):
        with pytest.raises(ValueError):
            ils.make_plan(*args)
    with pytest.raises(ValueError):
        ils.make_plan(4, 4, 1.0, 2.0, workers=0)
    with pytest.raises(ValueError):
        ils.SolverPlan(4, 4, 1.0, 2.0).with_data(np.zeros((5, 5)))


def test_as_plane_and_multiimage_validation():
    with pytest.raises(ValueError):
        ils.as_plane(np.zeros(3))
    with pytest.raises(ValueError):
        ils.as_plane(np.zeros((0, 3)))
    with pytest.raises(ValueError):
        ils.as_plane(np.array([[np.nan]]))
    with pytest.raises(ValueError):
        ils.MultiImage((np.zeros((2, 2)),), ils.RGB)
    img = ils.MultiImage.from_array(np.zeros((4, 5, 3)))
    assert img.height == 4 and img.width == 5 and img.space == ils.RGB
    assert not img.channels[0].flags.writeable


def test_energy_trace_contract():
    tr = ils.EnergyTrace([10.0, 6.0, 5.0, 4.0])
    assert tr.rel_decrease(1) == pytest.approx(4.0 / 6.0)
    assert tr.rel_decrease(3) == 1.0
    with pytest.raises(ValueError):
        tr.rel_decrease(4)
    with pytest.raises(ValueError):
        ils.EnergyTrace([]).rel_decrease(0)


def test_product_never_imports_the_oracle():
    pkg = os.path.join(ROOT, "paper_2003_07504_b200")
    for dirpath, _, files in os.walk(pkg):
        for fn in files:
            if fn.endswith(".py"):
                txt = open(os.path.join(dirpath, fn)).read()
                assert "oracle" not in re.sub(r"#.*|\"\"\"[\s\S]*?\"\"\"", "", txt), fn


def test_no_cpu_fallback_without_cuda():
    import torch

    if torch.cuda.is_available():
        pytest.skip("CUDA present")
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        ils.smooth_plane(np.zeros((8, 8)), ils.SmoothParams(ils.Charbonnier(0.8), 1.0))


def test_hqs_params_validation_matches_reference():
    # hqs.py:33-43 (HqsParams) and the C ABI's own checks (host-only plans, no GPU)
    import ctypes as C

    import paper_2003_07504_b200 as ils
    from paper_2003_07504_b200 import _lib

    for bad in (dict(lam=0.0), dict(lam=1.0, beta0=-1.0), dict(lam=1.0, kappa=1.0), dict(lam=1.0, iters=0)):
        with pytest.raises(ValueError):
            ils.HqsParams(**bad)
    assert ils.HqsParams(0.25).initial_beta == 0.5
    assert ils.HqsParams(0.25, beta0=3.0).initial_beta == 3.0
    L = _lib.lib()
    h = C.c_void_p()
    ok = _lib.HqsParams(0.25, 0.0, 2.0, 4)
    _lib.check(L.ils_hqs_plan_create(C.byref(h), 3, 1080, 1920, C.byref(ok), _lib.ILS_F32, -1), "create")
    L.ils_plan_destroy(h)
    for bad in (_lib.HqsParams(0.0, 0.0, 2.0, 4), _lib.HqsParams(1.0, -2.0, 2.0, 4), _lib.HqsParams(1.0, 0.0, 1.0, 4),
                _lib.HqsParams(1.0, 0.0, 2.0, 0), _lib.HqsParams(float("inf"), 0.0, 2.0, 4)):
        with pytest.raises(ValueError):
            _lib.check(L.ils_hqs_plan_create(C.byref(h), 1, 8, 8, C.byref(bad), _lib.ILS_F32, -1), "create")
    # the soft-threshold kind is not an ILS penalty: ils_plan_create refuses it
    p = _lib.Params(_lib.ILS_SOFT, 0.0, 0.0, 0.0, 1.0, 1.0, 4)
    with pytest.raises(ValueError):
        _lib.check(L.ils_plan_create(C.byref(h), 1, 8, 8, C.byref(p), _lib.ILS_F32, -1), "create")


def test_application_params_validation():
    # applications.py:23-77 (host-side, before any work)
    import paper_2003_07504_b200 as ils

    with pytest.raises(ValueError):
        ils.DetailBoost(-0.5)
    with pytest.raises(ValueError):
        ils.DetailBoost(float("inf"))
    assert ils.DetailBoost().k == 3.0
    base = ils.SmoothParams(ils.Charbonnier(1.0, 1e-4), 1.0)
    for kw in (dict(target_range=0.0), dict(saturation=0.0), dict(saturation=1.2), dict(log_offset=0.0),
               dict(lambdas=(1.0, 2.0)), dict(lambdas=(8.0, 1.0, 0.125)),
               dict(lambdas=(0.125, 1.0, 8.0), weights=(1.0, 1.0))):
        with pytest.raises(ValueError):
            ils.TonemapParams(base, **kw)
    ils.TonemapParams(base, lambdas=(1.0, 1.0, 1.0))


def test_bench_pass_order_matches_the_header():
    # include/ils_b200.h (ils_launch_pass): 0, 1, 2, 5, 6, 1, 2, 5, ..., ending with 3 or 7
    import importlib.util

    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(ROOT, "bench.py"))
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)
    assert bench.pass_order_of(4) == [0, 1, 2, 5, 6, 1, 2, 5, 7]
    assert bench.pass_order_of(1) == [0, 1, 3]
    assert bench.pass_order_of(3) == [0, 1, 2, 5, 6, 1, 3]
