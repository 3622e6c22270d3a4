"""CPU-side checks of the product library: it loads, exports every symbol the
public header declares, validates like the reference, plans pass geometry
like the reference, and refuses to compute without a GPU (no CPU fallback)."""
import ctypes as C
import os
import re

import numpy as np
import pytest

import paper_1705_01674_b200 as S
from paper_1705_01674_b200 import _native as N

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "sgwls_b200.h")


def header_symbols():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"\b(sgwls_b200_[a-z_]+)\s*\(", src)))


def test_header_symbols_exported():
    lib = C.CDLL(N.LIB_PATH)
    syms = header_symbols()
    assert len(syms) >= 12
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) <= set(N.SIGNATURES), set(syms) - set(N.SIGNATURES)


def test_library_is_sm100a():
    out = os.popen(f"cuobjdump -lelf {N.LIB_PATH} 2>/dev/null").read()
    if not out:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out


def test_defaults_match_reference():
    c = N.NativeConfig()
    N.lib().sgwls_b200_config_default(C.byref(c))
    d = S.SmoothConfig()
    assert (c.lambda_, c.r, c.tau, c.iterations, c.first_axis, c.threads) == (900.0, 1, 1, 4, 0, 1)
    assert (c.weight_kind, c.alpha_s, c.alpha_r, c.sigma_s, c.sigma_r, c.epsilon, c.guidance_scale) == \
        (0, 1.2, 1.2, 4.0, 3.0, 1e-4, 1.0)
    assert (d.lambda_, d.r, d.tau, d.iterations) == (900.0, 1, 1, 4)


@pytest.mark.parametrize("cfg,msg", [
    (S.SmoothConfig(lambda_=-1.0), "smooth: lambda must be finite and >= 0"),
    (S.SmoothConfig(lambda_=float("nan")), "smooth: lambda must be finite and >= 0"),
    (S.SmoothConfig(r=0), "smooth: r must be >= 1"),
    (S.SmoothConfig(r=2, tau=6), "smooth: tau must be in [1, 2r+1], got 6"),
    (S.SmoothConfig(tau=0), "smooth: tau must be in [1, 2r+1], got 0"),
    (S.SmoothConfig(iterations=0), "smooth: iterations must be >= 1"),
    (S.SmoothConfig(threads=0), "smooth: threads must be >= 1"),
    (S.SmoothConfig(weight=S.WeightParams(epsilon=0.0)), "weights: epsilon must be > 0"),
    (S.SmoothConfig(weight=S.WeightParams(kind=S.WeightKind.Exp, sigma_s=0.0)),
     "weights: sigma_s and sigma_r must be > 0 for exponential weights"),
    (S.SmoothConfig(weight=S.WeightParams(guidance_scale=-2.0)), "weights: guidance_scale must be > 0"),
])
def test_validation_texts(cfg, msg):
    with pytest.raises(S.Error) as e:
        S.validate(cfg)
    assert str(e.value) == msg


def test_validation_matches_oracle(port):
    from oracle.pyoracle import OracleError

    t = np.zeros((3, 3), np.float32)
    for cfg in [S.SmoothConfig(lambda_=-1.0), S.SmoothConfig(r=3, tau=8), S.SmoothConfig(iterations=-2)]:
        with pytest.raises(OracleError) as e1:
            port.smooth(t, t, cfg)
        with pytest.raises(S.Error) as e2:
            S.validate(cfg)
        assert str(e1.value) == str(e2.value)


def test_shape_errors():
    with pytest.raises(S.Error, match="smooth: target and guidance dimensions differ"):
        S.smooth(np.zeros((4, 4), np.float32), np.zeros((4, 5), np.float32))
    with pytest.raises(S.Error, match="smooth: empty target"):
        S.smooth(np.zeros((0, 4), np.float32), np.zeros((0, 4), np.float32))


def test_any_radius_validates_like_the_reference():
    """proj/src/smoother.cpp:105-107: every r >= 1 is valid (r > 8 runs the any-radius path)"""
    S.validate(S.SmoothConfig(r=9, tau=1))
    S.validate(S.SmoothConfig(r=40, tau=81))
    with pytest.raises(S.Error, match=r"smooth: tau must be in \[1, 2r\+1\], got 82"):
        S.validate(S.SmoothConfig(r=40, tau=82))


@pytest.mark.skipif(__import__("conftest").HAS_CUDA, reason="CPU-only check")
def test_no_cpu_fallback():
    with pytest.raises(S.CudaError, match="no CPU fallback"):
        S.smooth(np.zeros((4, 4), np.float32), np.zeros((4, 4), np.float32))


def _describe(extent, sweep, r, tau):
    info = np.zeros(6, dtype=np.int32)
    cap = extent + 4096
    cen = np.zeros(cap, dtype=np.int32)
    nb = N.lib().sgwls_b200_describe_pass(extent, sweep, r, tau, info.ctypes.data, cen.ctypes.data, cap)
    return nb, info, cen


@pytest.mark.parametrize("extent,r,tau", [(9, 1, 1), (9, 1, 3), (10, 1, 4), (2048, 3, 2), (1080, 1, 3),
                                          (1920, 1, 3), (8192, 2, 3), (1024, 2, 2), (512, 1, 1), (5, 3, 4),
                                          (1, 2, 3), (7, 3, 7), (3, 1, 3), (17, 8, 17)])
def test_band_centers_match_oracle(extent, r, tau, port):
    nb, info, cen = _describe(extent, 64, r, tau)
    want = port.band_centers(extent, r, tau)
    assert nb == len(want)
    assert cen[:nb].tolist() == want
    m = info[1]
    assert m == (2 * r + 1 if extent >= 2 * r + 1 else extent)


@pytest.mark.parametrize("extent,sweep,r,tau", [(1920, 1080, 1, 3), (1080, 1920, 1, 3), (2048, 2048, 3, 2),
                                                (8192, 8192, 2, 3), (1024, 1024, 2, 2), (1, 64, 2, 1),
                                                (64, 1, 2, 1), (3, 5, 3, 4), (40, 7, 8, 3)])
def test_chunking_invariants(extent, sweep, r, tau):
    """Every chunk holds >= 2r+1 positions (separators never couple directly)
    and the chunks tile the sweep exactly."""
    nb, info, cen = _describe(extent, sweep, r, tau)
    m, P, kmax = info[1], info[2], info[3]
    rows = cen[nb: nb + P + 1]
    assert rows[0] == 0 and rows[-1] == sweep
    sizes = np.diff(rows)
    assert (sizes > 0).all()
    if P > 1:
        assert (sizes * m >= 2 * r + 1).all()
    assert sizes.max() * m <= kmax


def test_kernel_launch_accounting():
    cfg = S.SmoothConfig(lambda_=400.0, r=1, tau=3, iterations=4)
    n = S.kernel_launches(1920, 1080, 3, 1, 1, False, cfg)
    assert n == 1 + 4 * 3  # guidance transpose + 4 passes x (KA, K2 tree, KB); r = 1 solves inner separators in KB
