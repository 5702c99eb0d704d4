"""The rolling-band row pass (csrc/ils_rowroll.cuh) against k_row (needs a B200).

For the 3840- and 7680-wide compile-time plans the first and fused row passes
run k_row_roll: a CTA walks a chunk of rows through a ring of line slots
instead of holding a band plus two recomputed halo rows.  The arithmetic is
k_row's, so the result must be bitwise identical to the k_row schedule
(ILS_NO_ROLL=1 at plan creation) for every chunk geometry, including chunks
that end in a partial step, chunks of one row and planes whose height is not
a multiple of the chunk; and within the north-star tolerance of the oracle
(test_gpu_parity.py: 4K Welsch, test_gpu_c5_columns.py: a full 8K plane).
"""

import ctypes as C

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs CUDA")]

import paper_2003_07504_b200 as ils  # noqa: E402
from paper_2003_07504_b200 import _lib  # noqa: E402
from paper_2003_07504_b200.penalty import params_of  # noqa: E402
from oracle import ils_oracle as O  # noqa: E402


def _smooth(f, params, monkeypatch, roll, rows=None, trace=False):
    """ils_smooth with a fresh plan built under the given schedule env."""
    monkeypatch.setenv("ILS_NO_ROLL", "0" if roll else "1")
    if rows:
        monkeypatch.setenv("ILS_ROLL_ROWS", str(rows))
    else:
        monkeypatch.delenv("ILS_ROLL_ROWS", raising=False)
    B, H, W = f.shape
    L = _lib.lib()
    h = C.c_void_p()
    _lib.check(L.ils_plan_create(C.byref(h), B, H, W, C.byref(params_of(params)), _lib.ILS_F32, 0))
    info = _lib.PlanInfo()
    L.ils_plan_get_info(h, C.byref(info))
    ws_sz = C.c_size_t()
    L.ils_workspace_size(h, C.byref(ws_sz))
    ws = torch.empty(ws_sz.value, dtype=torch.uint8, device="cuda")
    st = torch.empty(1, dtype=torch.int32, device="cuda")
    u = torch.empty_like(f)
    en = torch.empty((params.iters + 1, B), dtype=torch.float64, device="cuda") if trace else None
    _lib.check(L.ils_smooth(h, C.c_void_p(f.data_ptr()), C.c_void_p(u.data_ptr()), H * W, C.c_void_p(ws.data_ptr()),
                            C.c_void_p(torch.cuda.current_stream().cuda_stream), C.c_void_p(st.data_ptr()),
                            C.c_void_p(en.data_ptr()) if trace else None))
    torch.cuda.synchronize()
    L.ils_plan_destroy(h)
    return u, int(st.item()), info.row_roll_rows, en


@pytest.mark.parametrize("H,W,B,rows", [(2160, 3840, 3, None), (2160, 3840, 1, 7), (333, 3840, 2, 1),
                                        (4320, 7680, 1, None), (101, 7680, 1, 4), (64, 7680, 3, 64)])
def test_roll_bitwise_equals_k_row(H, W, B, rows, monkeypatch):
    params = ils.SmoothParams(ils.Welsch(10 / 255), 30.0, iters=4, c=2.0)
    f = torch.from_numpy(np.random.default_rng(H + W + B).random((B, H, W))).to("cuda", torch.float32)
    ur, sr, R, _ = _smooth(f, params, monkeypatch, True, rows)
    uk, sk, R0, _ = _smooth(f, params, monkeypatch, False)
    assert R > 0 and R0 == 0 and (rows is None or R == min(rows, H))
    assert sr == sk == _lib.STATUS_CLEAN
    assert torch.equal(ur, uk)


def test_roll_charbonnier_4k_matches_oracle(monkeypatch):
    params = ils.SmoothParams(ils.Charbonnier(0.8, 1e-4), 1.0, iters=4)
    f64 = np.random.default_rng(44).random((2160, 3840))
    u, st, R, _ = _smooth(torch.from_numpy(f64).to("cuda", torch.float32)[None], params, monkeypatch, True)
    assert R > 0 and st == _lib.STATUS_CLEAN
    ref = O.smooth_plane(f64, O.Charbonnier(0.8, 1e-4), 1.0, 4)
    assert np.max(np.abs(u[0].double().cpu().numpy() - ref)) <= 1e-4


def test_roll_flags_nonfinite_input_and_iterates(monkeypatch):
    params = ils.SmoothParams(ils.Charbonnier(0.8, 1e-4), 1.0, iters=3)
    f = torch.rand((1, 160, 3840), device="cuda")
    f[0, 77, 1234] = float("nan")
    _, st, R, _ = _smooth(f, params, monkeypatch, True, rows=16)
    assert R == 16 and st == 0  # non-finite input -> ValueError (image.py:43-44)
    huge = torch.full((1, 96, 7680), 1e30, device="cuda")
    huge[0, ::2, ::2] = -1e30
    big = ils.SmoothParams(ils.Charbonnier(0.8, 1e-4), 1e30, iters=3)
    _, st, R, _ = _smooth(huge, big, monkeypatch, True)
    assert R > 0 and 1 <= st <= 3  # the first non-finite iterate (smoother.py:166-167)


def test_traced_and_8bit_calls_keep_k_row_and_agree(monkeypatch):
    # energy traces and 8-bit ingest stay on k_row; their u equals the rolled one
    params = ils.SmoothParams(ils.Charbonnier(0.8, 1e-4), 1.0, iters=3)
    f = torch.rand((1, 120, 3840), device="cuda")
    ur, _, _, _ = _smooth(f, params, monkeypatch, True)
    ut, st, _, en = _smooth(f, params, monkeypatch, True, trace=True)
    assert st == _lib.STATUS_CLEAN and torch.equal(ur, ut)
    assert torch.all(en[1:] <= en[:-1] * (1 + 1e-6))


@pytest.mark.parametrize("H,W", [(333, 3840), (97, 7680)])
def test_final_pass_rows_per_cta_do_not_change_bits(H, W, monkeypatch):
    # the wide plans' final pass (c2r -> u, no halo) picks its own rows per CTA
    # (2 CTAs/SM); every choice must give the same bits
    params = ils.SmoothParams(ils.Welsch(10 / 255), 30.0, iters=3, c=2.0)
    f = torch.from_numpy(np.random.default_rng(H).random((2, H, W))).to("cuda", torch.float32)
    monkeypatch.delenv("ILS_FIN_BAND", raising=False)
    u0, s0, _, _ = _smooth(f, params, monkeypatch, True)
    assert s0 == _lib.STATUS_CLEAN
    for L in (1, 2, 3, 7):
        monkeypatch.setenv("ILS_FIN_BAND", str(L))
        u, s, _, _ = _smooth(f, params, monkeypatch, True)
        assert s == _lib.STATUS_CLEAN and torch.equal(u, u0), L
