"""Multi-GPU behind the C ABI (sgwls_b200_smooth_multi,
sgwls_b200_interpolate_sparse_batch_multi): one process drives the devices of
a list, the row-slab partitioned solve with slab records and halo rows moved
peer to peer.  The pool's boxes have one GPU, so several slabs share device 0
(the same code path: per-slab streams, buffers, peer copies and cross-device
event barriers); results must equal the single-device filter and the oracle.
A plain C++ caller (tests/cpp/multi_main.cpp) links the product library."""
import os
import subprocess

import numpy as np
import pytest

import paper_1705_01674_b200 as S
from paper_1705_01674_b200 import _native as N

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _img(h, w, c=1, seed=0):
    rng = np.random.default_rng(seed)
    base = rng.random((h // 8 + 1, w // 8 + 1, c)).repeat(8, 0).repeat(8, 1)[:h, :w]
    return np.clip(base + 0.05 * rng.standard_normal((h, w, c)), 0, 1).astype(np.float32)


def _cfg(r=2, tau=3, T=4, lam=400.0, fa=S.Axis.Column):
    return S.SmoothConfig(lambda_=lam, r=r, tau=tau, iterations=T, first_axis=fa,
                          weight=S.WeightParams(kind=S.WeightKind.Exp, sigma_r=0.05))


def test_multi_symbols_exported():
    for s in ("sgwls_b200_smooth_multi", "sgwls_b200_interpolate_sparse_batch_multi"):
        assert hasattr(N.lib(), s)


def test_multi_validates_before_touching_devices():
    t = np.zeros((8, 8), np.float32)
    with pytest.raises(S.Error, match="tau must be in"):
        S.smooth_multi(t, t, S.SmoothConfig(r=1, tau=5), devices=[0, 0])


@pytest.mark.gpu
@pytest.mark.parametrize("devs,cfg,shape", [
    ([0], _cfg(), (300, 257, 1)),
    ([0, 0], _cfg(), (300, 257, 1)),
    ([0, 0, 0], _cfg(r=1, tau=3, T=4), (270, 190, 3)),
    ([0, 0, 0, 0], _cfg(r=3, tau=2, T=3, lam=900.0), (256, 200, 1)),
    ([0, 0], _cfg(r=2, tau=2, T=4, fa=S.Axis.Row), (150, 170, 1)),
    ([0] * 8, _cfg(r=2, tau=3, T=2), (64, 140, 1)),
    ([0, 0], _cfg(r=6, tau=3, T=2), (80, 60, 1)),  # outside the slab mode: first device
])
def test_smooth_multi_matches_single_device(devs, cfg, shape, port):
    h, w, c = shape
    t = _img(h, w, c, seed=len(devs))
    g = _img(h, w, 1, seed=50 + len(devs))
    got = S.smooth_multi(t, g, cfg, devices=devs)
    one = S.smooth(t, g, cfg)
    want = port.smooth(t, g, cfg)
    d1 = float(np.abs(got - one).max())
    d2 = float(np.abs(got - want).max())
    print(f"smooth_multi {devs} {shape} r={cfg.r}: vs single device {d1:.2e}, vs oracle {d2:.2e}")
    assert d1 <= 2e-6 and d2 <= 1e-4


@pytest.mark.gpu
def test_smooth_multi_pivot_error(port):
    from oracle.pyoracle import OracleError

    t = _img(120, 90, 1, seed=1)
    g = _img(120, 90, 1, seed=2)
    g[77, 41, 0] = np.nan
    with pytest.raises(OracleError) as want:
        port.smooth(t, g, _cfg(T=2))
    with pytest.raises(S.Error) as got:
        S.smooth_multi(t, g, _cfg(T=2), devices=[0, 0, 0])
    assert str(got.value) == str(want.value)


@pytest.mark.gpu
def test_sparse_batch_multi_matches_batch():
    import ctypes as C

    rng = np.random.default_rng(3)
    b, h, w = 5, 64, 48
    g = rng.random((b, h, w)).astype(np.float32)
    m = (rng.random((b, h, w)) < 0.1).astype(np.float32)
    v = (m * rng.random((b, h, w))).astype(np.float32)
    cfg = _cfg(r=2, tau=2, T=4)
    want, wund = S.interpolate_sparse_batch(v, m, g, cfg)
    out = np.empty_like(v)
    und = np.empty_like(m)
    err = N.errbuf()
    devs = np.zeros(3, np.int32)
    rc = N.lib().sgwls_b200_interpolate_sparse_batch_multi(v.ctypes.data, m.ctypes.data, g.ctypes.data, b, w, h, 1,
                                                           1, C.byref(N.to_native(cfg)), devs.ctypes.data, 3,
                                                           out.ctypes.data, und.ctypes.data, err, len(err))
    N.check(rc, err)
    assert np.array_equal(out, want) and np.array_equal(und, wund)


@pytest.mark.gpu
@pytest.mark.parametrize("devs", ["0", "0,0", "0,0,0,0"])
def test_cpp_caller_smooth_multi(devs, tmp_path):
    exe = str(tmp_path / "multi_main")
    libdir = os.path.join(ROOT, "paper_1705_01674_b200")
    r = subprocess.run(["g++", "-O2", "-std=c++17", os.path.join(ROOT, "tests", "cpp", "multi_main.cpp"),
                        "-I" + os.path.join(ROOT, "include"), "-L" + libdir, "-l:libsgwls_b200.so",
                        "-Wl,-rpath," + libdir, "-o", exe], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    r = subprocess.run([exe, devs], capture_output=True, text=True, timeout=300)
    print(r.stdout.strip())
    assert r.returncode == 0, r.stdout + r.stderr
