"""The reference's application pipelines on the device (paper_1705_01674_b200.apps,
C ABI sgwls_b200_detail_enhance / _tone_map / _depth_upsample / _colorize)
against the reference's own apps.cpp (oracle/_ref/libsgwls_ref.so through
oracle.pyoracle.RefApps) on seeded synthetic inputs.

Bar: max |delta| relative to max(1, max |reference|) <= 1e-4, the filter's
own north-star tolerance (measured on B200: <= 6.2e-7 for every pipeline)."""
import os

import numpy as np
import pytest

import paper_1705_01674_b200 as S
from paper_1705_01674_b200 import apps as A

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HAVE_REF = os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libsgwls_ref.so"))
needs_ref = pytest.mark.skipif(not HAVE_REF, reason="reference library not built (needs /root/reference at build time)")


def _ref():
    from oracle.pyoracle import RefApps
    return RefApps()


def _rel(a, b):
    return float(np.abs(np.asarray(a, np.float64) - b).max()) / max(1.0, float(np.abs(b).max()))


def _blocks(h, w, seed):
    rng = np.random.default_rng(seed)
    y, x = np.mgrid[0:h, 0:w]
    img = 0.3 + 0.2 * (x > w * 0.4) + 0.25 * (y > h * 0.45) + 0.05 * ((x + y) % 3)
    return np.clip(img + rng.normal(0, 0.03, (h, w)), 0, 1).astype(np.float32)


def _scene(h, w, seed):
    """RGB guidance + piecewise-planar depth over the same regions."""
    rng = np.random.default_rng(seed)
    y, x = np.mgrid[0:h, 0:w]
    region = (x > w // 3).astype(int) + 2 * (y > h // 2)
    cols = rng.uniform(0.1, 0.9, (4, 3))
    rgb = np.clip(cols[region] + rng.normal(0, 0.01, (h, w, 3)), 0, 1).astype(np.float32)
    depth = (0.3 + 0.15 * region + 1e-3 * x - 5e-4 * y).astype(np.float32)
    return rgb, depth


# ------------------------------------------------------------ host (no GPU)

def test_presets_mirror_reference():
    """proj/src/apps.cpp:8-56"""
    e = A.enhance_preset()
    assert (e.lambda_, e.r, e.tau, e.iterations, e.weight.kind, e.weight.alpha_s, e.weight.alpha_r,
            e.weight.guidance_scale) == (900.0, 1, 1, 4, S.WeightKind.Frac, 1.2, 1.2, 1.0)
    t = A.tonemap_layer_preset(40.0)
    assert t.lambda_ == 40.0 and t.weight.kind == S.WeightKind.Frac and t.r == 1
    for f, lam in ((2, 100.0), (4, 200.0), (8, 400.0)):
        u = A.upsample_preset(f)
        assert (u.lambda_, u.r, u.tau, u.weight.kind, u.weight.sigma_s, u.weight.sigma_r,
                u.weight.guidance_scale) == (lam, 4, 4, S.WeightKind.Exp, 4.0, 3.0, 255.0)
    with pytest.raises(S.Error, match="upsample_preset: published lambdas cover factors 2, 4 and 8"):
        A.upsample_preset(3)
    c = A.colorize_preset()
    assert (c.lambda_, c.r, c.tau, c.weight.kind, c.weight.sigma_s, c.weight.sigma_r,
            c.weight.guidance_scale) == (900.0, 4, 2, S.WeightKind.Exp, 4.0, 2.0, 255.0)
    p = A.ToneMapParams()
    assert tuple(p.lambdas) == (5.0, 40.0, 320.0) and p.target_log_range == 2.0


@needs_ref
def test_input_errors_match_reference():
    """Checks that precede any device work carry the reference's texts."""
    from oracle.pyoracle import OracleError
    R = _ref()
    rgb, depth = _scene(32, 48, 1)
    low3 = np.ascontiguousarray(np.repeat(depth[::4, ::4, None], 3, axis=2))
    cases = [
        (lambda: A.depth_upsample(low3, rgb, 4, A.upsample_preset(4)),
         lambda: R.depth_upsample(low3, rgb, 4, A.upsample_preset(4))),
        (lambda: A.depth_upsample(depth[::4, ::4], rgb, 0, A.upsample_preset(4)),
         lambda: R.depth_upsample(depth[::4, ::4], rgb, 0, A.upsample_preset(4))),
        (lambda: A.depth_upsample(depth[::4, ::4], rgb[:, :40], 4, A.upsample_preset(4)),
         lambda: R.depth_upsample(depth[::4, ::4], rgb[:, :40], 4, A.upsample_preset(4))),
    ]
    for ours, ref in cases:
        with pytest.raises(OracleError) as e_ref:
            ref()
        with pytest.raises(S.Error) as e_ours:
            ours()
        assert str(e_ours.value) == str(e_ref.value)
    # sgwls::Image holds 1 or 3 channels (proj/src/image.cpp:14-16), so the
    # reference cannot build these inputs; luminance()'s own text is kept
    with pytest.raises(S.Error, match="luminance needs 1 or 3 channels"):
        A.tone_map(rgb[:, :, :2] + 0.1)
    with pytest.raises(S.Error, match="luminance needs 1 or 3 channels"):
        A.depth_upsample(depth[::4, ::4], rgb[:, :, :2], 4, A.upsample_preset(4))
    with pytest.raises(S.Error, match="colorize: gray image must be single-channel"):
        A.colorize(rgb, rgb, np.zeros((32, 48), np.float32), A.colorize_preset())
    with pytest.raises(S.Error, match="colorize: scribbles must be 3-channel"):
        A.colorize(rgb[:, :, 0], rgb[:, :, :2], np.zeros((32, 48), np.float32), A.colorize_preset())


# ------------------------------------------------------------ device parity

@pytest.mark.gpu
@needs_ref
@pytest.mark.parametrize("channels,iters", [(1, 2), (3, 4)])
def test_detail_enhance(channels, iters):
    img = _blocks(72, 96, 8)
    if channels == 3:
        img = np.stack([img, img[::-1, :], 1 - img], axis=2).astype(np.float32)
    cfg = A.enhance_preset().copy(iterations=iters)
    got = A.detail_enhance(img, 2.0, cfg)
    want = _ref().detail_enhance(img, 2.0, cfg)
    err = _rel(got, want)
    print(f"detail_enhance C={channels}: {err:.3g}")
    assert err <= 1e-4


@pytest.mark.gpu
@needs_ref
def test_tone_map():
    img = _blocks(60, 80, 9)
    y, x = np.mgrid[0:60, 0:80]
    hdr = np.stack([0.01 + img * (1 + 40 * (x > 40)) * (1 + 0.2 * c) for c in range(3)], axis=2).astype(np.float32)
    p = A.ToneMapParams()
    got = A.tone_map(hdr, p)
    want = _ref().tone_map(hdr, p)
    err = _rel(got, want)
    print(f"tone_map: {err:.3g}")
    assert err <= 1e-4
    p2 = A.ToneMapParams(lambdas=(2.0, 20.0, 200.0), detail_weights=(1.5, 1.0, 0.5), target_log_range=1.0)
    err2 = _rel(A.tone_map(hdr[:, :, 1], p2), _ref().tone_map(hdr[:, :, 1], p2))
    print(f"tone_map 1-channel, custom params: {err2:.3g}")
    assert err2 <= 1e-4


@pytest.mark.gpu
@needs_ref
def test_tone_map_rejects_nonpositive_luminance():
    hdr = np.full((16, 16, 3), 0.5, np.float32)
    hdr[3, 4] = 0.0
    with pytest.raises(S.Error, match="tone_map: luminance must be strictly positive"):
        A.tone_map(hdr)


@pytest.mark.gpu
@needs_ref
@pytest.mark.parametrize("factor", [2, 4])
def test_depth_upsample(factor):
    rgb, depth = _scene(64, 96, 11)
    low = np.ascontiguousarray(depth[::factor, ::factor])
    cfg = A.upsample_preset(factor)
    got = A.depth_upsample(low, rgb, factor, cfg)
    want = _ref().depth_upsample(low, rgb, factor, cfg)
    err = _rel(got, want)
    print(f"depth_upsample x{factor}: {err:.3g}")
    assert err <= 1e-4


@pytest.mark.gpu
@needs_ref
def test_colorize():
    rgb, _ = _scene(64, 96, 12)
    gray = (0.299 * rgb[..., 0] + 0.587 * rgb[..., 1] + 0.114 * rgb[..., 2]).astype(np.float32)
    scrib = np.zeros_like(rgb)
    mask = np.zeros(gray.shape, np.float32)
    mask[::7, ::5] = 1.0
    scrib[mask == 1] = rgb[mask == 1]
    cfg = A.colorize_preset()
    got = A.colorize(gray, scrib, mask, cfg)
    want = _ref().colorize(gray, scrib, mask, cfg)
    err = _rel(got, want)
    print(f"colorize: {err:.3g}")
    assert err <= 1e-4
    bad = mask.copy()
    bad[0, 0] = 0.5
    with pytest.raises(S.Error, match="interpolate_sparse: mask must be 0/1"):
        A.colorize(gray, scrib, bad, cfg)
    with pytest.raises(S.Error, match="interpolate_sparse: empty mask"):
        A.colorize(gray, scrib, np.zeros_like(mask), cfg)
