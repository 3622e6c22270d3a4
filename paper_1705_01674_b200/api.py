"""Python host mirror of the reference filter entry points.

``smooth`` mirrors ``sgwls::smooth`` (proj/include/sgwls/smoother.hpp:30,
proj/src/smoother.cpp:113-125) and ``interpolate_sparse`` mirrors
``sgwls::interpolate_sparse`` (proj/include/sgwls/smoother.hpp:41-42,
proj/src/smoother.cpp:127-163): same argument meaning, same defaults, same
``Error`` texts.  Images are numpy arrays of shape (H, W) or (H, W, C) holding
the row-major channel-interleaved samples of ``sgwls::Image``
(proj/include/sgwls/image.hpp:13-27); computation is fp32 on the GPU through
the C ABI.  The ``*_device`` forms take torch CUDA tensors and stay on the
device (stream-ordered, no host copies).
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native as N
from .config import Error, SmoothConfig, SparseField


def _as_hwc(a, name: str) -> np.ndarray:
    a = np.asarray(a)
    if a.ndim == 2:
        a = a[:, :, None]
    if a.ndim != 3:
        raise Error(f"{name}: expected an (H, W) or (H, W, C) image")
    return np.ascontiguousarray(a, dtype=np.float32)


def _check_same_size(t: np.ndarray, g: np.ndarray) -> None:
    if t.size == 0:
        raise Error("smooth: empty target")
    if t.shape[:2] != g.shape[:2]:
        raise Error("smooth: target and guidance dimensions differ")


def smooth(target, guidance, cfg: SmoothConfig | None = None) -> np.ndarray:
    """Edge-preserving SG-WLS smoothing of ``target`` under ``guidance``."""
    cfg = cfg or SmoothConfig()
    squeeze = np.asarray(target).ndim == 2
    t = _as_hwc(target, "smooth")
    g = _as_hwc(guidance, "smooth")
    _check_same_size(t, g)
    h, w, c = t.shape
    out = np.empty_like(t)
    err = N.errbuf()
    nc = N.to_native(cfg)
    rc = N.lib().sgwls_b200_smooth(t.ctypes.data, w, h, c, g.ctypes.data, g.shape[2], C.byref(nc),
                                   out.ctypes.data, err, len(err))
    N.check(rc, err)
    return out[:, :, 0] if squeeze else out


def smooth_batch(targets, guidances, cfg: SmoothConfig | None = None) -> np.ndarray:
    """``len(targets)`` independent ``smooth`` calls, (B, H, W[, C]) arrays."""
    cfg = cfg or SmoothConfig()
    t = np.ascontiguousarray(targets, dtype=np.float32)
    g = np.ascontiguousarray(guidances, dtype=np.float32)
    squeeze = t.ndim == 3
    if squeeze:
        t = t[..., None]
    if g.ndim == 3:
        g = g[..., None]
    b, h, w, c = t.shape
    out = np.empty_like(t)
    err = N.errbuf()
    nc = N.to_native(cfg)
    rc = N.lib().sgwls_b200_smooth_batch(t.ctypes.data, g.ctypes.data, b, w, h, c, g.shape[3], C.byref(nc),
                                         out.ctypes.data, err, len(err))
    N.check(rc, err)
    return out[..., 0] if squeeze else out


def smooth_multi(target, guidance, cfg: SmoothConfig | None = None, devices=None) -> np.ndarray:
    """``smooth`` of ONE image in row slabs over several GPUs of this process
    (``sgwls_b200_smooth_multi``: slab records all-gathered, halos exchanged peer
    to peer).  devices: CUDA ordinals, one per slab (repeats allowed); None = the
    SGWLS_B200_DEVICES list, else device 0."""
    cfg = cfg or SmoothConfig()
    squeeze = np.asarray(target).ndim == 2
    t = _as_hwc(target, "smooth")
    g = _as_hwc(guidance, "smooth")
    _check_same_size(t, g)
    h, w, c = t.shape
    out = np.empty_like(t)
    err = N.errbuf()
    nc = N.to_native(cfg)
    devs = np.ascontiguousarray(devices if devices is not None else [], dtype=np.int32)
    rc = N.lib().sgwls_b200_smooth_multi(t.ctypes.data, w, h, c, g.ctypes.data, g.shape[2], C.byref(nc),
                                         devs.ctypes.data if devs.size else None, int(devs.size), out.ctypes.data,
                                         err, len(err))
    N.check(rc, err)
    return out[:, :, 0] if squeeze else out


def interpolate_sparse(field: SparseField, guidance, cfg: SmoothConfig | None = None,
                       return_undefined: bool = False):
    """Guided interpolation smooth(values)/smooth(mask) (Eq. 21)."""
    cfg = cfg or SmoothConfig()
    squeeze = np.asarray(field.values).ndim == 2
    v = _as_hwc(field.values, "interpolate_sparse")
    m = np.asarray(field.mask)
    if m.ndim == 3:
        if m.shape[2] != 1:
            raise Error("interpolate_sparse: mask must be single-channel")
        m = m[:, :, 0]
    m = np.ascontiguousarray(m, dtype=np.float32)
    if m.shape != v.shape[:2]:
        raise Error("interpolate_sparse: values/mask size mismatch")
    # field checks before smooth()'s own (proj/src/smoother.cpp:129-147): the
    # first offending pixel in scan order decides the text
    bad01 = (m != 0) & (m != 1)
    offv = (m == 0) & np.any(v != 0, axis=2)
    both = bad01 | offv
    if both.any():
        k = int(np.argmax(both.ravel()))
        raise Error("interpolate_sparse: mask must be 0/1" if bad01.ravel()[k]
                    else "interpolate_sparse: values nonzero outside mask")
    if not (m == 1).any():
        raise Error("interpolate_sparse: empty mask")
    validate(cfg)
    g = _as_hwc(guidance, "interpolate_sparse")
    if v.size == 0:
        raise Error("smooth: empty target")
    if g.shape[:2] != v.shape[:2]:
        raise Error("smooth: target and guidance dimensions differ")
    h, w, c = v.shape
    out = np.empty_like(v)
    und = np.empty((h, w), dtype=np.float32)
    err = N.errbuf()
    nc = N.to_native(cfg)
    rc = N.lib().sgwls_b200_interpolate_sparse(v.ctypes.data, m.ctypes.data, w, h, c, g.ctypes.data, g.shape[2],
                                               C.byref(nc), out.ctypes.data, und.ctypes.data, err, len(err))
    N.check(rc, err)
    res = out[:, :, 0] if squeeze else out
    return (res, und) if return_undefined else res


def interpolate_sparse_batch(values, masks, guidances, cfg: SmoothConfig | None = None):
    """Batched interpolate_sparse over (B, H, W) values / masks / guidances; returns (out, undefined)."""
    cfg = cfg or SmoothConfig()
    v = np.ascontiguousarray(values, dtype=np.float32)
    m = np.ascontiguousarray(masks, dtype=np.float32)
    g = np.ascontiguousarray(guidances, dtype=np.float32)
    b, h, w = v.shape[:3]
    c = v.shape[3] if v.ndim == 4 else 1
    gc = g.shape[3] if g.ndim == 4 else 1
    out = np.empty_like(v)
    und = np.empty((b, h, w), dtype=np.float32)
    err = N.errbuf()
    nc = N.to_native(cfg)
    rc = N.lib().sgwls_b200_interpolate_sparse_batch(v.ctypes.data, m.ctypes.data, g.ctypes.data, b, w, h, c, gc,
                                                     C.byref(nc), out.ctypes.data, und.ctypes.data, err, len(err))
    N.check(rc, err)
    return out, und


# ------------------------------------------------------------ device forms

def _stream_ptr(stream, device) -> int:
    """Raw handle of ``stream`` (default: the current stream of ``device``); the
    stream must belong to the tensors' device."""
    import torch

    s = stream if stream is not None else torch.cuda.current_stream(device)
    if s.device != device:
        raise Error(f"sgwls_b200: stream is on {s.device}, tensors are on {device}")
    return int(s.cuda_stream)


def _dev_dims(t, name):
    """(B, H, W, C) of a contiguous fp32 CUDA tensor shaped (H,W), (H,W,C) or (B,H,W,C)."""
    import torch

    if not isinstance(t, torch.Tensor) or not (t.is_cuda and t.dtype == torch.float32 and t.is_contiguous()):
        raise Error(f"{name}: expected a contiguous float32 CUDA tensor")
    if t.dim() == 2:
        return 1, t.shape[0], t.shape[1], 1
    if t.dim() == 3:
        return 1, t.shape[0], t.shape[1], t.shape[2]
    if t.dim() == 4:
        return tuple(t.shape)
    raise Error(f"{name}: bad tensor rank")


def _same_device(name, ref, *ts):
    for t in ts:
        if t is not None and t.device != ref.device:
            raise Error(f"{name}: all tensors must be on {ref.device} (got {t.device})")


def _check_out(t, shape, ref, name):
    """A caller-supplied output must be a contiguous fp32 tensor of exactly
    ``shape`` on the inputs' device (the kernels write through a raw pointer)."""
    import torch

    if not isinstance(t, torch.Tensor) or not (t.is_cuda and t.dtype == torch.float32 and t.is_contiguous()):
        raise Error(f"{name}: expected a contiguous float32 CUDA tensor")
    if tuple(t.shape) != tuple(shape):
        raise Error(f"{name}: expected shape {tuple(shape)}, got {tuple(t.shape)}")
    _same_device(name, ref, t)


def smooth_device(target, guidance, cfg: SmoothConfig | None = None, out=None, stream=None, sync: bool = False,
                  graph: bool = False):
    """smooth on torch CUDA tensors, (H,W[,C]) or batched (B,H,W,C); stream-ordered.
    graph=True captures the call into a CUDA graph once per (buffers, shape, config) and replays it.
    The kernels run on the tensors' device (made current for the call)."""
    import torch

    cfg = cfg or SmoothConfig()
    b, h, w, c = _dev_dims(target, "smooth")
    bg, hg, wg, gc = _dev_dims(guidance, "smooth")
    if (hg, wg) != (h, w) or bg != b:
        raise Error("smooth: target and guidance dimensions differ")
    _same_device("smooth", target, guidance)
    if out is None:
        out = torch.empty_like(target)
    else:
        _check_out(out, target.shape, target, "smooth: out")
    err = N.errbuf()
    nc = N.to_native(cfg)
    flags = (N.SYNC if sync else 0) | (N.GRAPH if graph else 0)
    with torch.cuda.device(target.device):
        rc = N.lib().sgwls_b200_smooth_device(target.data_ptr(), guidance.data_ptr(), b, w, h, c, gc, C.byref(nc),
                                              out.data_ptr(), _stream_ptr(stream, target.device), flags, err,
                                              len(err))
    N.check(rc, err)
    return out


def pass_device(src, guidance, cfg: SmoothConfig | None = None, out=None, stream=None, sync: bool = False,
                graph: bool = False):
    """ONE Column-axis pass (proj/src/smoother.cpp:51-99) on torch CUDA tensors (H,W[,C]) or (B,H,W,C),
    written transposed: returns (W,H[,C]) / (B,W,H,C).  cfg.iterations / cfg.first_axis are ignored."""
    import torch

    cfg = cfg or SmoothConfig()
    b, h, w, c = _dev_dims(src, "pass")
    bg, hg, wg, gc = _dev_dims(guidance, "pass")
    if (hg, wg) != (h, w) or bg != b:
        raise Error("smooth: target and guidance dimensions differ")
    _same_device("pass", src, guidance)
    shape = (w, h) if src.dim() == 2 else ((w, h, c) if src.dim() == 3 else (b, w, h, c))
    if out is None:
        out = torch.empty(shape, dtype=torch.float32, device=src.device)
    else:
        _check_out(out, shape, src, "pass: out")
    err = N.errbuf()
    nc = N.to_native(cfg)
    flags = (N.SYNC if sync else 0) | (N.GRAPH if graph else 0)
    with torch.cuda.device(src.device):
        rc = N.lib().sgwls_b200_pass_device(src.data_ptr(), guidance.data_ptr(), b, w, h, c, gc, C.byref(nc),
                                            out.data_ptr(), _stream_ptr(stream, src.device), flags, err, len(err))
    N.check(rc, err)
    return out


def interpolate_sparse_device(values, masks, guidances, cfg: SmoothConfig | None = None, out=None,
                              undefined=None, stream=None, sync: bool = False, validate: bool = False,
                              graph: bool = False):
    """Batched interpolate_sparse on torch CUDA tensors: values (B,H,W) or (B,H,W,C), masks (B,H,W),
    guidances (B,H,W) or (B,H,W,Cg); out like values, undefined (B,H,W).  Stream-ordered.
    validate=True runs the reference's field checks (mask 0/1, values zero off the mask, non-empty
    mask) on the device for every pair, with one host synchronisation."""
    import torch

    cfg = cfg or SmoothConfig()
    for t, nm in ((values, "values"), (masks, "masks"), (guidances, "guidances")):
        _dev_dims(t, f"interpolate_sparse: {nm}")
    if values.dim() == 3:
        b, h, w = values.shape
        c = 1
    elif values.dim() == 4:
        b, h, w, c = values.shape
    else:
        raise Error("interpolate_sparse: values must be (B,H,W) or (B,H,W,C)")
    if masks.dim() != 3 or tuple(masks.shape) != (b, h, w):
        raise Error("interpolate_sparse: values/mask size mismatch")
    if guidances.dim() == 3:
        gshape, gc = tuple(guidances.shape), 1
    elif guidances.dim() == 4:
        gshape, gc = tuple(guidances.shape[:3]), guidances.shape[3]
    else:
        raise Error("interpolate_sparse: guidances must be (B,H,W) or (B,H,W,Cg)")
    if gshape != (b, h, w):
        raise Error("smooth: target and guidance dimensions differ")
    _same_device("interpolate_sparse", values, masks, guidances)
    if out is None:
        out = torch.empty_like(values)
    else:
        _check_out(out, values.shape, values, "interpolate_sparse: out")
    if undefined is not None:
        _check_out(undefined, (b, h, w), values, "interpolate_sparse: undefined")
    und_ptr = undefined.data_ptr() if undefined is not None else None
    err = N.errbuf()
    nc = N.to_native(cfg)
    flags = (N.SYNC if sync else 0) | (N.VALIDATE if validate else 0) | (N.GRAPH if graph else 0)
    with torch.cuda.device(values.device):
        rc = N.lib().sgwls_b200_interpolate_sparse_device(values.data_ptr(), masks.data_ptr(), guidances.data_ptr(),
                                                          b, w, h, c, gc, C.byref(nc), out.data_ptr(), und_ptr,
                                                          _stream_ptr(stream, values.device), flags, err, len(err))
    N.check(rc, err)
    return out


def validate(cfg: SmoothConfig) -> None:
    """SmoothConfig::validate (proj/src/smoother.cpp:103-111)."""
    err = N.errbuf()
    nc = N.to_native(cfg)
    N.check(N.lib().sgwls_b200_validate(C.byref(nc), err, len(err)), err)


def kernel_launches(width, height, channels, guidance_channels, batch, sparse, cfg: SmoothConfig) -> int:
    nc = N.to_native(cfg)
    return int(N.lib().sgwls_b200_kernel_launches(width, height, channels, guidance_channels, batch,
                                                  1 if sparse else 0, C.byref(nc)))


def graph_clear() -> int:
    """Release every cached CUDA graph of graph=True calls (waits for their last replay)."""
    return int(N.lib().sgwls_b200_graph_clear())


def graph_count() -> int:
    return int(N.lib().sgwls_b200_graph_count())


def version() -> str:
    return N.lib().sgwls_b200_version().decode()


def read_image(path: str) -> np.ndarray:
    """sgwls::read_image (proj/include/sgwls/image.hpp:41): PGM/PPM scaled to [0,1] or PFM,
    as an (H, W, C) float32 array; decode failures carry the reference's byte-offset text."""
    data = C.POINTER(C.c_float)()
    w, h, c = C.c_int(), C.c_int(), C.c_int()
    err = N.errbuf()
    N.check(N.lib().sgwls_b200_image_read(str(path).encode(), C.byref(data), C.byref(w), C.byref(h), C.byref(c),
                                          err, len(err)), err)
    try:
        return np.ctypeslib.as_array(data, shape=(h.value, w.value, c.value)).copy()
    finally:
        N.lib().sgwls_b200_image_free(data)


def write_image(img, path: str) -> None:
    """sgwls::write_image (proj/include/sgwls/image.hpp:46): .pgm / .ppm (clamped, 8-bit,
    round half up) or .pfm by extension."""
    a = np.asarray(img, dtype=np.float32)
    if a.ndim == 2:
        a = a[:, :, None]
    a = np.ascontiguousarray(a)
    err = N.errbuf()
    ptr = a.ctypes.data_as(C.c_void_p) if a.size else None
    h, w, c = (a.shape if a.ndim == 3 else (0, 0, 0))
    N.check(N.lib().sgwls_b200_image_write(str(path).encode(), ptr, w, h, c, err, len(err)), err)
