"""Host mirror of the reference's application pipelines (proj/include/sgwls/apps.hpp,
proj/src/apps.cpp): ``detail_enhance``, ``tone_map``, ``depth_upsample``,
``colorize`` and the four parameter presets, same argument meaning, defaults and
``Error`` texts.  Every stage runs on the GPU through the C ABI
(``sgwls_b200_detail_enhance`` ... in include/sgwls_b200.h): one upload, the
filter passes and the elementwise stages on device buffers, one download.
Images are numpy arrays (H, W) or (H, W, C) as in ``api.smooth``.
"""
from __future__ import annotations

import ctypes as C
import dataclasses

import numpy as np

from . import _native as N
from .api import _as_hwc
from .config import Error, SmoothConfig


def _preset(fn, *args) -> SmoothConfig:
    nc = N.NativeConfig()
    fn(*args, C.byref(nc))
    return N.from_native(nc)


def enhance_preset() -> SmoothConfig:
    """frac, alpha_s = alpha_r = 1.2, lambda = 900, r = 1, tau = 1 (proj/src/apps.cpp:8-20)"""
    return _preset(N.lib().sgwls_b200_enhance_preset)


def tonemap_layer_preset(lambda_: float) -> SmoothConfig:
    """enhance_preset with the given lambda (proj/src/apps.cpp:22-26)"""
    return _preset(N.lib().sgwls_b200_tonemap_layer_preset, float(lambda_))


def upsample_preset(factor: int) -> SmoothConfig:
    """exp, sigma_s = 4, sigma_r = 3, r = 4, tau = 4, lambda 100/200/400 for factor 2/4/8 (proj/src/apps.cpp:28-44)"""
    nc = N.NativeConfig()
    err = N.errbuf()
    N.check(N.lib().sgwls_b200_upsample_preset(int(factor), C.byref(nc), err, len(err)), err)
    return N.from_native(nc)


def colorize_preset() -> SmoothConfig:
    """exp, sigma_s = 4, sigma_r = 2, r = 4, tau = 2, lambda = 900 (proj/src/apps.cpp:46-56)"""
    return _preset(N.lib().sgwls_b200_colorize_preset)


@dataclasses.dataclass
class ToneMapParams:
    """proj/include/sgwls/apps.hpp:21-30"""
    lambdas: tuple = (5.0, 40.0, 320.0)
    detail_weights: tuple = (1.0, 1.0, 1.0)
    target_log_range: float = 2.0
    smoothing: SmoothConfig = dataclasses.field(default_factory=lambda: tonemap_layer_preset(5.0))


def _out(shape, squeeze):
    out = np.empty(shape, dtype=np.float32)
    return out, (lambda a: a[:, :, 0] if squeeze else a)


def detail_enhance(img, boost: float, cfg: SmoothConfig) -> np.ndarray:
    """clamp(base + boost*(img - base), 0, 1) with base = smooth(img, img, cfg) (proj/src/apps.cpp:58-64)"""
    squeeze = np.asarray(img).ndim == 2
    a = _as_hwc(img, "detail_enhance")
    h, w, c = a.shape
    out, fin = _out(a.shape, squeeze)
    err = N.errbuf()
    nc = N.to_native(cfg)
    N.check(N.lib().sgwls_b200_detail_enhance(a.ctypes.data, w, h, c, float(boost), C.byref(nc), out.ctypes.data,
                                              err, len(err)), err)
    return fin(out)


def tone_map(hdr, params: ToneMapParams | None = None) -> np.ndarray:
    """Three-level log-luminance decomposition, base compression, chroma reattachment (proj/src/apps.cpp:66-109)"""
    params = params or ToneMapParams()
    squeeze = np.asarray(hdr).ndim == 2
    a = _as_hwc(hdr, "tone_map")
    h, w, c = a.shape
    p = N.NativeToneMapParams()
    for i in range(3):
        p.lambdas[i] = float(params.lambdas[i])
        p.detail_weights[i] = float(params.detail_weights[i])
    p.target_log_range = float(params.target_log_range)
    p.smoothing = N.to_native(params.smoothing)
    out, fin = _out(a.shape, squeeze)
    err = N.errbuf()
    N.check(N.lib().sgwls_b200_tone_map(a.ctypes.data, w, h, c, C.byref(p), out.ctypes.data, err, len(err)), err)
    return fin(out)


def depth_upsample(lowres_depth, guidance, factor: int, cfg: SmoothConfig) -> np.ndarray:
    """Project the low-resolution depth to (y*factor, x*factor), guided sparse interpolation
    under the guidance's luma (proj/src/apps.cpp:111-128).  Returns (H, W)."""
    d = _as_hwc(lowres_depth, "depth_upsample")
    g = _as_hwc(guidance, "depth_upsample")
    out = np.empty(g.shape[:2], dtype=np.float32)
    err = N.errbuf()
    nc = N.to_native(cfg)
    N.check(N.lib().sgwls_b200_depth_upsample(d.ctypes.data, d.shape[1], d.shape[0], d.shape[2], g.ctypes.data,
                                              g.shape[1], g.shape[0], g.shape[2], int(factor), C.byref(nc),
                                              out.ctypes.data, err, len(err)), err)
    return out


def colorize(gray, scribbles, scribble_mask, cfg: SmoothConfig) -> np.ndarray:
    """Propagate the scribbles' U, V over the gray image; Y = gray (proj/src/apps.cpp:130-155).  Returns (H, W, 3)."""
    g = _as_hwc(gray, "colorize")
    s = _as_hwc(scribbles, "colorize")
    m = _as_hwc(scribble_mask, "colorize")
    if g.shape[2] != 1:
        raise Error("colorize: gray image must be single-channel")
    if s.shape[2] != 3:
        raise Error("colorize: scribbles must be 3-channel")
    if g.shape[:2] != s.shape[:2] or g.shape[:2] != m.shape[:2]:
        raise Error("colorize: image sizes differ")
    if m.shape[2] != 1:
        raise Error("interpolate_sparse: mask must be single-channel")
    h, w = g.shape[:2]
    out = np.empty((h, w, 3), dtype=np.float32)
    err = N.errbuf()
    nc = N.to_native(cfg)
    N.check(N.lib().sgwls_b200_colorize(g.ctypes.data, 1, s.ctypes.data, 3, m.ctypes.data, w, h, C.byref(nc),
                                        out.ctypes.data, err, len(err)), err)
    return out
