"""Pin the CPU oracle (oracle/sgwls_oracle.c) before trusting it.

1. Against the golden fixtures produced by the reference library itself
   (tests/golden/make_golden.py) -- these run everywhere, incl. the GPU box.
2. Against the reference library live (oracle/_ref), where it is built.
3. Against the SPEC.md worked examples.
All comparisons are bit-exact: the restatement keeps the reference's
operation order.
"""
import json
import os

import numpy as np
import pytest

from paper_1705_01674_b200.config import Axis, SmoothConfig, WeightKind, WeightParams

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "golden.npz")


def _cfg(case, threads=1):
    h, w, c, cg, lam, r, tau, T, kind, axis, sr, gs = case
    return SmoothConfig(lambda_=lam, r=r, tau=tau, iterations=T,
                        weight=WeightParams(kind=WeightKind(kind), sigma_r=sr, guidance_scale=gs),
                        first_axis=Axis(axis), threads=threads)


@pytest.fixture(scope="module")
def golden():
    z = np.load(GOLDEN)
    meta = json.loads(bytes(z["meta"]).decode())
    return z, meta


def test_golden_smooth(golden, port):
    z, meta = golden
    for i, case in enumerate(meta["smooth"]):
        got = port.smooth(z[f"smooth{i}_t"], z[f"smooth{i}_g"], _cfg(case))
        assert np.array_equal(got, z[f"smooth{i}_out"]), f"case {i} {case}"


def test_golden_smooth_threads(golden, port):
    """proj/include/sgwls/smoother.hpp:19-21: bit-identical for any thread count."""
    z, meta = golden
    for i, case in enumerate(meta["smooth"]):
        got = port.smooth(z[f"smooth{i}_t"], z[f"smooth{i}_g"], _cfg(case, threads=4))
        assert np.array_equal(got, z[f"smooth{i}_out"])


def test_golden_sparse(golden, port):
    z, meta = golden
    for i, case in enumerate(meta["sparse"]):
        o, und = port.interpolate_sparse(z[f"sparse{i}_v"], z[f"sparse{i}_m"], z[f"sparse{i}_g"], _cfg(case))
        assert np.array_equal(o, z[f"sparse{i}_out"])
        assert np.array_equal(und, z[f"sparse{i}_und"])


def test_golden_band_solves(golden, port):
    z, meta = golden
    for i, (n, r, lam) in enumerate(meta["band"]):
        u, alpha, beta, gamma = port.solve_band(z[f"band{i}_w"], lam, z[f"band{i}_rhs"], r)
        rb = min(r, n - 1)
        assert np.array_equal(u, z[f"band{i}_u"])
        assert np.array_equal(alpha, z[f"band{i}_alpha"])
        assert np.array_equal(beta[: n * rb], z[f"band{i}_beta"][: n * rb])
        assert np.array_equal(gamma[: n * rb], z[f"band{i}_gamma"][: n * rb])


def test_golden_centers(golden, port):
    _, meta = golden
    for ext, r, tau, want in meta["centers"]:
        assert port.band_centers(ext, r, tau) == want


def test_spec_tridiagonal_example(port):
    """[[2,-1,0],[-1,3,-1],[0,-1,2]], f=[1,2,3]."""
    u, alpha, beta, gamma = port.solve_band(np.array([1.0, 1.0, 0.0]), 1.0, np.array([1.0, 2.0, 3.0]), 1)
    assert np.allclose(alpha, [2.0, 2.5, 1.6], atol=1e-15)
    assert np.allclose(beta[:2], [-0.5, -0.4], atol=1e-15)
    assert np.allclose(gamma[:2], [-1.0, -1.0], atol=1e-15)
    assert np.allclose(u, [1.5, 2.0, 2.5], atol=1e-15)


def test_spec_band_centers(port):
    """SPEC.md:278-280 (1-indexed there, 0-indexed here)."""
    assert port.band_centers(9, 1, 1) == [1, 2, 3, 4, 5, 6, 7]
    assert port.band_centers(9, 1, 3) == [1, 4, 7]
    assert port.band_centers(10, 1, 4) == [1, 5, 8]


def test_spec_serpentine(port):
    """3x3 image, r=1, column mode, centre 1 -> [1,2,3,6,5,4,7,8,9]."""
    img = np.arange(1, 10, dtype=np.float64).reshape(3, 3)
    rows, cols = port.band_layout(3, 3, 1, 1, 0)
    assert img[rows, cols].tolist() == [1, 2, 3, 6, 5, 4, 7, 8, 9]


def test_port_matches_reference_live(ref, port):
    rng = np.random.default_rng(77)
    for trial in range(25):
        h, w = int(rng.integers(1, 40)), int(rng.integers(1, 40))
        r = int(rng.integers(1, 6))
        tau = int(rng.integers(1, 2 * r + 2))
        c = int(rng.choice([1, 3]))
        cg = int(rng.choice([1, 3]))
        case = (h, w, c, cg, float(rng.choice([0.0, 5.0, 400.0, 900.0])), r, tau, int(rng.integers(1, 5)),
                int(rng.integers(0, 2)), int(rng.integers(0, 2)), float(rng.choice([0.05, 0.3, 3.0])),
                float(rng.choice([1.0, 255.0])))
        t = rng.uniform(0, 1, (h, w, c)).astype(np.float32)
        g = rng.uniform(0, 1, (h, w, cg)).astype(np.float32)
        a = port.smooth(t, g, _cfg(case))
        b = ref.smooth(t, g, _cfg(case))
        assert np.array_equal(a, b), case


def test_port_matches_reference_weights(ref, port):
    rng = np.random.default_rng(78)
    g = rng.uniform(0, 1, (13, 11, 3))
    for kind in (0, 1):
        cfg = SmoothConfig(weight=WeightParams(kind=WeightKind(kind), sigma_r=0.2, guidance_scale=2.0))
        for axis in (0, 1):
            for center, r in [(0, 2), (5, 1), (10, 3), (6, 4)]:
                a = port.edge_weights(g, center, r, axis, cfg)
                b = ref.edge_weights(g, center, r, axis, cfg)
                assert np.array_equal(a, b)


def test_error_texts_match_reference(ref, port):
    from oracle.pyoracle import OracleError

    t = np.zeros((4, 4), np.float32)
    bad = [SmoothConfig(lambda_=-1.0), SmoothConfig(r=0), SmoothConfig(tau=4), SmoothConfig(iterations=0),
           SmoothConfig(threads=0), SmoothConfig(weight=WeightParams(epsilon=0.0)),
           SmoothConfig(weight=WeightParams(kind=WeightKind.Exp, sigma_r=0.0)),
           SmoothConfig(weight=WeightParams(guidance_scale=0.0)), SmoothConfig(lambda_=float("inf"))]
    for cfg in bad:
        with pytest.raises(OracleError) as e1:
            port.smooth(t, t, cfg)
        with pytest.raises(OracleError) as e2:
            ref.smooth(t, t, cfg)
        assert str(e1.value) == str(e2.value)


def test_sparse_errors_match_reference(ref, port):
    from oracle.pyoracle import OracleError

    g = np.ones((6, 6), np.float32)
    cases = []
    m = np.zeros((6, 6), np.float32)
    cases.append((np.zeros((6, 6), np.float32), m.copy()))
    m2 = m.copy()
    m2[1, 2] = 0.5
    cases.append((np.zeros((6, 6), np.float32), m2))
    m3 = m.copy()
    m3[3, 3] = 1
    v3 = np.zeros((6, 6), np.float32)
    v3[0, 1] = 2.0
    cases.append((v3, m3))
    for v, mm in cases:
        with pytest.raises(OracleError) as e1:
            port.interpolate_sparse(v, mm, g, SmoothConfig())
        with pytest.raises(OracleError) as e2:
            ref.interpolate_sparse(v, mm, g, SmoothConfig())
        assert str(e1.value) == str(e2.value)


def test_nan_guidance_error_matches_reference(ref, port):
    from oracle.pyoracle import OracleError

    rng = np.random.default_rng(3)
    t = rng.uniform(0, 1, (10, 12)).astype(np.float32)
    g = t.copy()
    g[4, 7] = np.nan
    cfg = SmoothConfig(lambda_=400.0, r=2, tau=2, weight=WeightParams(kind=WeightKind.Exp, sigma_r=0.1))
    with pytest.raises(OracleError) as e1:
        port.smooth(t, g, cfg)
    with pytest.raises(OracleError) as e2:
        ref.smooth(t, g, cfg)
    assert str(e1.value) == str(e2.value)
    assert "non-positive pivot at row" in str(e1.value)
