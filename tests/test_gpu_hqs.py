"""HQS penalty-splitting baseline on the GPU vs the reference.

Goldens: tests/golden/golden.npz hqs_* (the real hqs_smooth_plane, hqs.py:50-66).
Larger sizes: the oracle's restatement (tests/test_oracle_golden.py pins it).
"""

import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2003_07504_b200 as ils  # noqa: E402
from oracle import ils_oracle as O  # noqa: E402

GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def g():
    return np.load(os.path.join(GOLD, "golden.npz"))


def _params(arr):
    lam, beta0, kappa, iters = arr
    return ils.HqsParams(float(lam), beta0=None if beta0 < 0 else float(beta0), kappa=float(kappa), iters=int(iters))


@pytest.mark.parametrize("prec", ["fp64", "fp32"])
def test_hqs_matches_reference_goldens(g, prec):
    names = sorted({k[:-4] for k in g.files if k.startswith("hqs_") and k.endswith("_prm")})
    assert len(names) == 5
    for name in names:
        u = ils.hqs_smooth_plane(g[name + "_f"], _params(g[name + "_prm"]), precision=prec)
        ref = g[name + "_u"]
        err = float(np.max(np.abs(u - ref)))
        if prec == "fp64":
            assert err < 1e-10, (name, err)  # test_hqs.py:80 holds the CPU path to 1e-13
        else:
            assert err <= 1e-4 and O.psnr(u, ref) >= 60.0, (name, err)


def test_hqs_1080p_rgb_batch_matches_oracle():
    rng = np.random.default_rng(20240607)
    f = rng.random((3, 1080, 1920))
    prm = ils.HqsParams(0.05, iters=4)
    u = ils.hqs_smooth_batch(torch.from_numpy(f).to("cuda", torch.float32), prm).double().cpu().numpy()
    for c in range(3):
        ref = O.hqs_smooth_plane(f[c], 0.05, iters=4, workers=8)
        err = float(np.max(np.abs(u[c] - ref)))
        assert err <= 1e-4 and O.psnr(u[c], ref) >= 60.0, (c, err)
    # a plane smoothed alone equals it inside the batch, bit for bit
    one = ils.hqs_smooth_plane(torch.from_numpy(f[1]).to("cuda", torch.float32), prm)
    assert np.array_equal(one.double().cpu().numpy(), u[1])


def test_hqs_behaviour_matches_reference_tests():
    # pkg/tests/test_hqs.py:86-109 on the GPU path
    rng = np.random.default_rng(3)
    f = np.clip(0.5 + 0.25 * np.cumsum(rng.standard_normal((32, 32)), axis=1) / 6, 0, 1)
    a = ils.hqs_smooth_plane(f, ils.HqsParams(0.25), precision="fp64")
    b = ils.smooth_plane(f, ils.SmoothParams(ils.Charbonnier(1.0, 1e-4), 0.25), precision="fp64")
    assert np.max(np.abs(a - b)) > 1e-3
    assert np.max(np.abs(a - f)) > 1e-4
    rng = np.random.default_rng(4)
    clean = np.full((32, 32), 0.25)
    clean[:, 16:] = 0.75
    noisy = np.clip(clean + 0.05 * rng.standard_normal((32, 32)), 0.0, 1.0)
    out = ils.hqs_smooth_plane(noisy, ils.HqsParams(0.25))
    assert np.mean((out - clean) ** 2) < np.mean((noisy - clean) ** 2) / 2


def test_hqs_rejects_bad_input_and_trace():
    with pytest.raises(ValueError):
        ils.hqs_smooth_plane(np.full((8, 8), np.nan), ils.HqsParams(0.25))
    with pytest.raises(ValueError):
        ils.hqs_smooth_plane(np.zeros((8, 8)), ils.HqsParams(0.25), workers=0)
    from paper_2003_07504_b200 import _runtime as rt

    with pytest.raises(ValueError, match="energy trace"):
        rt.smooth_device(torch.zeros((1, 8, 8), device="cuda"), ils.HqsParams(0.25).c_params(), trace=True)
