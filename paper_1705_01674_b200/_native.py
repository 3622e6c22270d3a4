"""ctypes binding of the native C ABI (include/sgwls_b200.h).

The library is the product: there is no Python or CPU fallback.  If
``libsgwls_b200.so`` is missing, importing the compute API raises.
"""
from __future__ import annotations

import ctypes as C
import os

from .config import Axis, CudaError, Error, SmoothConfig, WeightKind

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SGWLS_B200_LIB") or os.path.join(PKG, "libsgwls_b200.so")

OK, EINVAL, ECUDA, EUNSUPPORTED = 0, 1, 2, 3
SYNC, VALIDATE, GRAPH = 1, 2, 4


class NativeConfig(C.Structure):
    """sgwls_b200_config (include/sgwls_b200.h)"""
    _fields_ = [
        ("lambda_", C.c_double),
        ("r", C.c_int),
        ("tau", C.c_int),
        ("iterations", C.c_int),
        ("first_axis", C.c_int),
        ("threads", C.c_int),
        ("weight_kind", C.c_int),
        ("alpha_s", C.c_double),
        ("alpha_r", C.c_double),
        ("sigma_s", C.c_double),
        ("sigma_r", C.c_double),
        ("epsilon", C.c_double),
        ("guidance_scale", C.c_double),
    ]


class NativeToneMapParams(C.Structure):
    """sgwls_b200_tonemap_params (include/sgwls_b200.h), ToneMapParams proj/include/sgwls/apps.hpp:21-30"""
    _fields_ = [
        ("lambdas", C.c_double * 3),
        ("detail_weights", C.c_double * 3),
        ("target_log_range", C.c_double),
        ("smoothing", NativeConfig),
    ]


def from_native(n: NativeConfig) -> SmoothConfig:
    from .config import WeightParams
    return SmoothConfig(lambda_=n.lambda_, r=n.r, tau=n.tau, iterations=n.iterations,
                        weight=WeightParams(kind=WeightKind(n.weight_kind), alpha_s=n.alpha_s, alpha_r=n.alpha_r,
                                            sigma_s=n.sigma_s, sigma_r=n.sigma_r, epsilon=n.epsilon,
                                            guidance_scale=n.guidance_scale),
                        first_axis=Axis(n.first_axis), threads=n.threads)


def to_native(cfg: SmoothConfig) -> NativeConfig:
    w = cfg.weight
    return NativeConfig(float(cfg.lambda_), int(cfg.r), int(cfg.tau), int(cfg.iterations),
                        int(Axis(cfg.first_axis)), int(cfg.threads), int(WeightKind(w.kind)),
                        float(w.alpha_s), float(w.alpha_r), float(w.sigma_s), float(w.sigma_r),
                        float(w.epsilon), float(w.guidance_scale))


_P = C.c_void_p
_lib = None

# exported symbols and their signatures; tests check that every symbol the
# header declares is present
SIGNATURES = {
    "sgwls_b200_config_default": (None, [C.POINTER(NativeConfig)]),
    "sgwls_b200_validate": (C.c_int, [C.POINTER(NativeConfig), C.c_char_p, C.c_size_t]),
    "sgwls_b200_smooth": (C.c_int, [_P, C.c_int, C.c_int, C.c_int, _P, C.c_int, C.POINTER(NativeConfig), _P,
                                    C.c_char_p, C.c_size_t]),
    "sgwls_b200_smooth_batch": (C.c_int, [_P, _P, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                          C.POINTER(NativeConfig), _P, C.c_char_p, C.c_size_t]),
    "sgwls_b200_smooth_device": (C.c_int, [_P, _P, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                           C.POINTER(NativeConfig), _P, _P, C.c_int, C.c_char_p, C.c_size_t]),
    "sgwls_b200_pass_device": (C.c_int, [_P, _P, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                         C.POINTER(NativeConfig), _P, _P, C.c_int, C.c_char_p, C.c_size_t]),
    "sgwls_b200_interpolate_sparse": (C.c_int, [_P, _P, C.c_int, C.c_int, C.c_int, _P, C.c_int,
                                                C.POINTER(NativeConfig), _P, _P, C.c_char_p, C.c_size_t]),
    "sgwls_b200_interpolate_sparse_batch": (C.c_int, [_P, _P, _P, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                                      C.POINTER(NativeConfig), _P, _P, C.c_char_p, C.c_size_t]),
    "sgwls_b200_interpolate_sparse_device": (C.c_int, [_P, _P, _P, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                                       C.POINTER(NativeConfig), _P, _P, _P, C.c_int, C.c_char_p,
                                                       C.c_size_t]),
    "sgwls_b200_kernel_launches": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                             C.POINTER(NativeConfig)]),
    "sgwls_b200_describe_pass": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, _P, _P, C.c_int]),
    "sgwls_b200_profile": (None, [C.c_int]),
    "sgwls_b200_profile_read": (C.c_int, [C.c_char_p, C.c_size_t]),
    "sgwls_b200_profile_collect": (None, []),
    "sgwls_b200_version": (C.c_char_p, []),
    "sgwls_b200_graph_clear": (C.c_int, []),
    "sgwls_b200_graph_count": (C.c_int, []),
    "sgwls_b200_transpose_device": (C.c_int, [_P, _P, C.c_int, C.c_int, C.c_int, C.c_int, _P, C.c_char_p,
                                              C.c_size_t]),
    # row-slab mode (slabs.py)
    "sgwls_b200_slab_sizes": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(NativeConfig),
                                        C.POINTER(C.c_size_t), C.POINTER(C.c_size_t), C.c_char_p, C.c_size_t]),
    "sgwls_b200_slab_pass_a": (C.c_int, [_P, _P, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                         C.POINTER(NativeConfig), _P, _P, _P, C.c_char_p, C.c_size_t]),
    "sgwls_b200_slab_pass_b": (C.c_int, [_P, _P, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                         C.POINTER(NativeConfig), _P, _P, _P, _P, _P, C.c_char_p, C.c_size_t]),
    # multi-GPU, one process
    "sgwls_b200_smooth_multi": (C.c_int, [_P, C.c_int, C.c_int, C.c_int, _P, C.c_int, C.POINTER(NativeConfig), _P,
                                          C.c_int, _P, C.c_char_p, C.c_size_t]),
    "sgwls_b200_interpolate_sparse_batch_multi": (C.c_int, [_P, _P, _P, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                                            C.POINTER(NativeConfig), _P, C.c_int, _P, _P, C.c_char_p,
                                                            C.c_size_t]),
    # image files (proj/src/image.cpp:111-250)
    "sgwls_b200_image_read": (C.c_int, [C.c_char_p, C.POINTER(C.POINTER(C.c_float)), C.POINTER(C.c_int),
                                        C.POINTER(C.c_int), C.POINTER(C.c_int), C.c_char_p, C.c_size_t]),
    "sgwls_b200_image_free": (None, [C.POINTER(C.c_float)]),
    "sgwls_b200_image_write": (C.c_int, [C.c_char_p, _P, C.c_int, C.c_int, C.c_int, C.c_char_p, C.c_size_t]),
    # application pipelines (proj/src/apps.cpp)
    "sgwls_b200_enhance_preset": (None, [C.POINTER(NativeConfig)]),
    "sgwls_b200_tonemap_layer_preset": (None, [C.c_double, C.POINTER(NativeConfig)]),
    "sgwls_b200_upsample_preset": (C.c_int, [C.c_int, C.POINTER(NativeConfig), C.c_char_p, C.c_size_t]),
    "sgwls_b200_colorize_preset": (None, [C.POINTER(NativeConfig)]),
    "sgwls_b200_tonemap_params_default": (None, [C.POINTER(NativeToneMapParams)]),
    "sgwls_b200_detail_enhance": (C.c_int, [_P, C.c_int, C.c_int, C.c_int, C.c_double, C.POINTER(NativeConfig), _P,
                                            C.c_char_p, C.c_size_t]),
    "sgwls_b200_tone_map": (C.c_int, [_P, C.c_int, C.c_int, C.c_int, C.POINTER(NativeToneMapParams), _P,
                                      C.c_char_p, C.c_size_t]),
    "sgwls_b200_depth_upsample": (C.c_int, [_P, C.c_int, C.c_int, C.c_int, _P, C.c_int, C.c_int, C.c_int, C.c_int,
                                            C.POINTER(NativeConfig), _P, C.c_char_p, C.c_size_t]),
    "sgwls_b200_colorize": (C.c_int, [_P, C.c_int, _P, C.c_int, _P, C.c_int, C.c_int, C.POINTER(NativeConfig), _P,
                                      C.c_char_p, C.c_size_t]),
}


def lib():
    """Load libsgwls_b200.so once; raises ImportError if it has not been built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() "
                              "(the SG-WLS path has no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def check(rc: int, err) -> None:
    if rc == OK:
        return
    msg = err.value.decode(errors="replace")
    if rc == ECUDA:
        raise CudaError(msg)
    raise Error(msg)


def errbuf():
    return C.create_string_buffer(1024)
