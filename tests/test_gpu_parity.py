"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Bar (BASELINE.json north_star): max |delta| <= 1e-4 on [0,1]-scaled fp32
intensities against the reference algorithm on the same fp32 inputs.  The
oracle is the C restatement (oracle/sgwls_oracle.c), itself pinned to the
reference library and the golden fixtures by tests/test_oracle.py.
"""
import os

import numpy as np
import pytest

import paper_1705_01674_b200 as S
from paper_1705_01674_b200 import workloads as WL

TOL = 1e-4
NTHREADS = os.cpu_count() or 1

pytestmark = pytest.mark.gpu


def _cfg(lam, r, tau, T, kind, axis, sigma_r=0.1, gscale=1.0):
    return S.SmoothConfig(lambda_=lam, r=r, tau=tau, iterations=T,
                          weight=S.WeightParams(kind=S.WeightKind(kind), sigma_r=sigma_r, guidance_scale=gscale),
                          first_axis=S.Axis(axis), threads=NTHREADS)


def _piecewise(rng, h, w, c, cells=6):
    """blocky random guidance: realistic edges + noise"""
    ys = np.sort(rng.integers(0, max(1, h), cells))
    xs = np.sort(rng.integers(0, max(1, w), cells))
    lab = (np.searchsorted(ys, np.arange(h))[:, None] * (cells + 1) + np.searchsorted(xs, np.arange(w))[None, :])
    vals = rng.uniform(0, 1, ((cells + 1) ** 2, c))
    img = vals[lab] + rng.normal(0, 0.02, (h, w, c))
    return img.astype(np.float32)


CASES = [
    # (h, w, c, cg, lam, r, tau, T, kind, axis)
    (17, 23, 1, 1, 400.0, 1, 1, 4, 1, 0),
    (40, 31, 3, 1, 400.0, 1, 3, 4, 1, 0),
    (40, 31, 3, 3, 900.0, 2, 2, 4, 0, 1),
    (64, 1, 1, 1, 50.0, 2, 1, 1, 1, 1),
    (1, 64, 1, 1, 50.0, 2, 1, 1, 1, 1),
    (1, 64, 1, 1, 50.0, 2, 1, 2, 1, 0),
    (5, 3, 1, 3, 300.0, 3, 4, 2, 0, 0),
    (2, 2, 1, 1, 300.0, 4, 9, 4, 1, 0),
    (1, 1, 1, 1, 300.0, 2, 3, 4, 1, 0),
    (33, 65, 2, 1, 900.0, 3, 2, 4, 1, 0),
    (100, 80, 1, 1, 400.0, 2, 3, 3, 1, 1),
    (97, 203, 1, 1, 900.0, 3, 7, 4, 0, 0),
    (120, 90, 4, 2, 100.0, 4, 4, 4, 1, 0),
    (150, 64, 1, 1, 0.0, 2, 2, 4, 1, 0),
    (70, 70, 1, 1, 1.0, 5, 6, 2, 1, 1),
    (60, 45, 1, 1, 400.0, 6, 3, 2, 1, 0),
    (60, 45, 1, 1, 400.0, 7, 15, 2, 0, 1),
    (80, 50, 1, 1, 400.0, 8, 8, 2, 1, 0),
    (300, 257, 1, 1, 900.0, 1, 1, 4, 1, 0),
    (257, 300, 3, 1, 400.0, 2, 5, 4, 1, 1),
    # r > 8: the any-radius path (sgwls_anyr.cu); the reference takes every r >= 1
    (60, 70, 1, 1, 400.0, 9, 5, 2, 1, 0),
    (50, 90, 3, 3, 900.0, 12, 25, 3, 0, 1),
    (40, 45, 2, 1, 200.0, 20, 7, 2, 1, 0),   # one axis clipped (45 < 2r+1 on neither, 40 < 41 on the row pass)
    (9, 30, 1, 1, 300.0, 16, 33, 4, 1, 0),   # both extents below 2r+1: single clipped bands
    (64, 100, 1, 2, 100.0, 10, 1, 1, 0, 1),
]


@pytest.mark.parametrize("case", CASES, ids=[f"{c[0]}x{c[1]}x{c[2]}_r{c[5]}t{c[6]}T{c[7]}k{c[8]}a{c[9]}"
                                              for c in CASES])
def test_smooth_matches_oracle(case, port):
    h, w, c, cg, lam, r, tau, T, kind, axis = case
    rng = np.random.default_rng(hash(case) % (2 ** 32))
    t = _piecewise(rng, h, w, c)
    g = _piecewise(rng, h, w, cg)
    cfg = _cfg(lam, r, tau, T, kind, axis)
    want = port.smooth(t, g, cfg)
    got = S.smooth(t, g, cfg)
    err = np.abs(got.astype(np.float64) - want).max()
    assert err <= TOL, f"max|d|={err:.3g}"


def test_interpolate_sparse_matches_oracle(port):
    rng = np.random.default_rng(5)
    h, w = 90, 70
    g = _piecewise(rng, h, w, 1)[:, :, 0]
    mask = (rng.uniform(0, 1, (h, w)) < 1 / 16).astype(np.float32)
    vals = np.where(mask > 0, rng.uniform(0.2, 1, (h, w)), 0).astype(np.float32)
    cfg = _cfg(400.0, 2, 2, 4, 1, 0, sigma_r=0.05)
    want, wund = port.interpolate_sparse(vals, mask, g, cfg)
    got, gund = S.interpolate_sparse(S.SparseField(vals, mask), g, cfg, return_undefined=True)
    assert np.abs(got - want).max() <= TOL
    assert (gund == wund).all()


SPARSE_CASES = [
    # (h, w, C values, r, tau, T, first axis): first pass reads values + mask
    # unpacked and the last pass writes the ratio (tiled path), or the pack /
    # ratio kernels (first axis Row: pack; clipped geometry: generic path)
    (90, 70, 1, 2, 2, 4, 0),
    (90, 70, 2, 1, 3, 3, 0),   # last pass a column pass: ratio untransposed
    (64, 80, 3, 4, 2, 1, 0),   # T = 1: split input and ratio in the same pass
    (75, 66, 1, 2, 3, 4, 1),   # first axis Row: packed input, fused ratio
    (40, 4, 1, 2, 1, 2, 0),    # width < 2r+1: generic path, pack + ratio kernels
]


@pytest.mark.parametrize("case", SPARSE_CASES, ids=[f"{c[0]}x{c[1]}c{c[2]}_r{c[3]}t{c[4]}T{c[5]}a{c[6]}"
                                                    for c in SPARSE_CASES])
def test_interpolate_sparse_paths(case, port):
    import torch

    h, w, c, r, tau, T, fa = case
    rng = np.random.default_rng(sum(case))
    g = _piecewise(rng, h, w, 1)[:, :, 0]
    mask = (rng.uniform(0, 1, (h, w)) < 1 / 8).astype(np.float32)
    mask[0, 0] = 1.0
    vals = (mask[:, :, None] * rng.uniform(0.2, 1, (h, w, c))).astype(np.float32)
    cfg = _cfg(400.0, r, tau, T, 1, fa, sigma_r=0.05)
    want, wund = port.interpolate_sparse(vals, mask, g, cfg)
    got, gund = S.interpolate_sparse(S.SparseField(vals, mask), g, cfg, return_undefined=True)
    assert np.abs(got - want.reshape(got.shape)).max() <= TOL
    assert (gund == wund).all()
    # device batch form (2 pairs) = host form, bit for bit
    dv = torch.from_numpy(np.stack([vals, vals])).cuda()
    dm = torch.from_numpy(np.stack([mask, mask])).cuda()
    dg = torch.from_numpy(np.stack([g, g])).cuda()
    und = torch.empty_like(dm)
    out = S.interpolate_sparse_device(dv, dm, dg, cfg, undefined=und, validate=True, sync=True)
    assert np.array_equal(out[1].cpu().numpy(), got.reshape(h, w, c))
    assert np.array_equal(und[0].cpu().numpy(), gund)


def test_batch_equals_single():
    rng = np.random.default_rng(9)
    ts = np.stack([_piecewise(rng, 50, 40, 1)[:, :, 0] for _ in range(3)])
    gs = np.stack([_piecewise(rng, 50, 40, 1)[:, :, 0] for _ in range(3)])
    cfg = _cfg(400.0, 2, 2, 4, 1, 0)
    batch = S.smooth_batch(ts, gs, cfg)
    for i in range(3):
        single = S.smooth(ts[i], gs[i], cfg)
        assert np.array_equal(batch[i], single)


def test_deterministic():
    rng = np.random.default_rng(11)
    t = _piecewise(rng, 130, 110, 3)
    g = _piecewise(rng, 130, 110, 1)
    cfg = _cfg(900.0, 3, 2, 4, 1, 0)
    a = S.smooth(t, g, cfg)
    b = S.smooth(t, g, cfg)
    assert np.array_equal(a, b)


def test_constant_invariance():
    rng = np.random.default_rng(12)
    g = _piecewise(rng, 77, 91, 1)
    for r, tau in [(1, 1), (2, 3), (3, 2), (4, 4)]:
        cfg = _cfg(900.0, r, tau, 4, 0, 0)
        out = S.smooth(np.full((77, 91), 0.625, np.float32), g, cfg)
        assert np.abs(out - 0.625).max() <= 1e-6


def test_lambda_zero_identity():
    rng = np.random.default_rng(13)
    t = rng.uniform(0, 1, (45, 38)).astype(np.float32)
    out = S.smooth(t, t, _cfg(0.0, 2, 2, 4, 1, 0))
    assert np.abs(out - t).max() <= 1e-6


def test_nan_guidance_reports_pivot(port):
    rng = np.random.default_rng(14)
    t = rng.uniform(0, 1, (20, 16)).astype(np.float32)
    g = t.copy()
    g[7, 9] = np.nan
    cfg = _cfg(400.0, 1, 1, 2, 1, 0)
    from oracle.pyoracle import OracleError
    with pytest.raises(OracleError) as oe:
        port.smooth(t, g, cfg)
    with pytest.raises(S.Error) as ge:
        S.smooth(t, g, cfg)
    assert str(ge.value) == str(oe.value)


def test_sparse_validation_errors():
    g = np.ones((8, 8), np.float32)
    m = np.zeros((8, 8), np.float32)
    v = np.zeros((8, 8), np.float32)
    with pytest.raises(S.Error, match="interpolate_sparse: empty mask"):
        S.interpolate_sparse(S.SparseField(v, m), g)
    m[2, 3] = 0.5
    with pytest.raises(S.Error, match="interpolate_sparse: mask must be 0/1"):
        S.interpolate_sparse(S.SparseField(v, m), g)
    m[2, 3] = 0.0
    m[1, 1] = 1.0
    v[0, 5] = 0.3
    with pytest.raises(S.Error, match="interpolate_sparse: values nonzero outside mask"):
        S.interpolate_sparse(S.SparseField(v, m), g)


def test_device_api_matches_host():
    import torch

    rng = np.random.default_rng(15)
    t = _piecewise(rng, 64, 48, 3)
    g = _piecewise(rng, 64, 48, 1)
    cfg = _cfg(400.0, 1, 3, 4, 1, 0)
    host = S.smooth(t, g, cfg)
    dt = torch.from_numpy(t).cuda()
    dg = torch.from_numpy(g).cuda()
    out = S.smooth_device(dt, dg, cfg, sync=True)
    assert np.array_equal(out.cpu().numpy(), host)


def test_graph_replay_matches_direct():
    import torch

    rng = np.random.default_rng(16)
    t = torch.from_numpy(_piecewise(rng, 130, 90, 3)).cuda()
    g = torch.from_numpy(_piecewise(rng, 130, 90, 1)).cuda()
    cfg = _cfg(400.0, 2, 3, 4, 1, 0)
    direct = S.smooth_device(t, g, cfg, sync=True)
    out = torch.empty_like(t)
    for _ in range(3):  # capture, then replays
        out.zero_()
        S.smooth_device(t, g, cfg, out=out, graph=True, sync=True)
        assert torch.equal(out, direct)
    t.mul_(0.5)  # same buffers, new contents: the replay must see them
    S.smooth_device(t, g, cfg, out=out, graph=True, sync=True)
    assert torch.equal(out, S.smooth_device(t, g, cfg, sync=True))


# ------------------------------------------------ BASELINE configurations

def _full(name, port, max_images=None, secondary=False):
    wl = WL.workload(name, secondary=secondary)
    cfg = wl.cfg.copy(threads=NTHREADS)
    gen = WL.GENERATORS[name]
    if wl.sparse:
        errs = []
        for i in range(max_images or 1):
            v, m, g = gen(i)
            want, wund = port.interpolate_sparse(v, m, g, cfg)
            got, gund = S.interpolate_sparse(S.SparseField(v, m), g, cfg, return_undefined=True)
            errs.append(np.abs(got - want).max())
            assert (gund == wund).all()
        return max(errs)
    t, g = gen(0)
    want = port.smooth(t, g, cfg)
    got = S.smooth(t, g, cfg)
    return np.abs(got.astype(np.float64) - want).max()


@pytest.mark.slow
@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c4"])
def test_baseline_config_parity(name, port):
    err = _full(name, port, max_images=2)
    print(f"{name}: max|d| = {err:.3g}")
    assert err <= TOL


@pytest.mark.slow
def test_baseline_c5_parity(port):
    err = _full("c5", port)
    print(f"c5: max|d| = {err:.3g}")
    assert err <= TOL


@pytest.mark.slow
@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c4", "c5"])
def test_baseline_secondary_reading_parity(name, port):
    """SURVEY.md 8(d) secondary reading: iterations = tau sweeps at stride 1."""
    err = _full(name, port, max_images=1, secondary=True)
    print(f"{name} (iterations = tau, tau = 1): max|d| = {err:.3g}")
    assert err <= TOL


@pytest.mark.slow
def test_c4_batch_parity_16_pairs(port):
    """c4 through the batched device path the bench times: 16 of the 64 pairs
    (every 4th) in ONE interpolate_sparse_device call, each pair against the
    oracle, with the reference's field validation on the device."""
    import torch

    wl = WL.workload("c4")
    cfg = wl.cfg.copy(threads=NTHREADS)
    ids = list(range(0, 64, 4))
    trip = [WL.gen_c4(i) for i in ids]
    dv, dm, dg = (torch.from_numpy(np.stack([t[k] for t in trip])).cuda() for k in range(3))
    und = torch.empty_like(dm)
    out = S.interpolate_sparse_device(dv, dm, dg, cfg, undefined=und, validate=True, sync=True)
    out, und = out.cpu().numpy(), und.cpu().numpy()
    worst = 0.0
    for k, (v, m, g) in enumerate(trip):
        want, wund = port.interpolate_sparse(v, m, g, cfg)
        worst = max(worst, float(np.abs(out[k] - want.reshape(out[k].shape)).max()))
        assert (und[k] == wund).all(), ids[k]
    print(f"c4 pairs {ids}: max|d| = {worst:.3g}")
    assert worst <= TOL


def test_any_radius_sparse_and_pivot_error(port):
    """r > 8 through interpolate_sparse (pack / ratio kernels around the any-radius passes)
    and the reference's pivot failure on NaN guidance"""
    rng = np.random.default_rng(99)
    h, w = 48, 56
    g = _piecewise(rng, h, w, 1)[:, :, 0]
    mask = (rng.uniform(size=(h, w)) < 0.1).astype(np.float32)
    vals = (_piecewise(rng, h, w, 1)[:, :, 0] * mask).astype(np.float32)
    cfg = _cfg(300.0, 10, 6, 2, 1, 0)
    want, und_w = port.interpolate_sparse(vals, mask, g, cfg)
    got, und = S.interpolate_sparse(S.SparseField(vals, mask), g, cfg, return_undefined=True)
    assert np.abs(got.astype(np.float64) - want.reshape(got.shape)).max() <= TOL
    assert np.array_equal(und.reshape(und_w.shape) != 0, und_w != 0)
    gbad = g.copy()
    gbad[20, 30] = np.nan
    with pytest.raises(S.Error, match="non-positive pivot"):
        S.smooth(vals, gbad, cfg)


def test_random_shapes_on_the_staged_path(port):
    """Seeded random r = 2 cases with rows on 16-byte bounds in both orientations: KB's TMA-staged
    input (tensor-map boxes starting off the 16-byte grid, partial last row tiles, first / interior /
    last band tiles, 1-3 channels, both first axes) against the oracle."""
    rng = np.random.default_rng(20261021)
    worst = 0.0
    for i in range(14):
        h = 4 * int(rng.integers(10, 120))
        w = 4 * int(rng.integers(10, 130))
        c = int(rng.integers(1, 4))
        tau = int(rng.integers(1, 6))
        T = int(rng.integers(1, 5))
        axis = int(rng.integers(0, 2))
        kind = int(rng.integers(0, 2))
        t = _piecewise(rng, h, w, c)
        g = _piecewise(rng, h, w, 1)
        cfg = _cfg(float(rng.choice([50.0, 400.0, 900.0])), 2, tau, T, kind, axis)
        err = float(np.abs(S.smooth(t, g, cfg).astype(np.float64) - port.smooth(t, g, cfg)).max())
        worst = max(worst, err)
        assert err <= TOL, f"case {i}: {h}x{w}x{c} tau={tau} T={T} axis={axis} kind={kind}: max|d|={err:.3g}"
    print(f"staged random shapes: worst max|d| = {worst:.3g}")
