"""Input checks of the host API in the reference's order (CPU, no device
needed: every case fails before a kernel would run).

proj/src/smoother.cpp:127-147: interpolate_sparse checks the mask channels,
the values/mask size, then scans the field (first offending pixel decides
between "mask must be 0/1" and "values nonzero outside mask"), then "empty
mask", and only then smooth()'s own checks (configuration, empty target,
guidance size)."""
import ctypes as C

import numpy as np
import pytest

import paper_1705_01674_b200 as S
from paper_1705_01674_b200 import _native as N


def _field(h=6, w=8):
    return np.zeros((h, w), np.float32), np.zeros((h, w), np.float32)


def test_sparse_bad_mask_before_guidance_size():
    v, m = _field()
    m[2, 3] = 0.5
    v[4, 4] = 1.0  # a later fault of the other kind
    with pytest.raises(S.Error) as e:
        S.interpolate_sparse(S.SparseField(v, m), np.zeros((6, 9), np.float32))
    assert str(e.value) == "interpolate_sparse: mask must be 0/1"


def test_sparse_first_fault_in_scan_order():
    v, m = _field()
    v[1, 1] = 2.0   # off-mask value first in scan order
    m[3, 3] = 7.0   # bad mask value later
    with pytest.raises(S.Error) as e:
        S.interpolate_sparse(S.SparseField(v, m), np.zeros((6, 8), np.float32))
    assert str(e.value) == "interpolate_sparse: values nonzero outside mask"


def test_sparse_field_before_config():
    v, m = _field()
    m[0, 0] = 1.0
    v[1, 1] = 2.0
    with pytest.raises(S.Error) as e:
        S.interpolate_sparse(S.SparseField(v, m), np.zeros((6, 8), np.float32), S.SmoothConfig(r=0))
    assert str(e.value) == "interpolate_sparse: values nonzero outside mask"


def test_sparse_empty_mask_before_config_and_size():
    v, m = _field()
    with pytest.raises(S.Error) as e:
        S.interpolate_sparse(S.SparseField(v, m), np.zeros((6, 9), np.float32), S.SmoothConfig(r=0))
    assert str(e.value) == "interpolate_sparse: empty mask"


def test_sparse_config_before_guidance_size():
    v, m = _field()
    m[0, 0] = 1.0
    with pytest.raises(S.Error) as e:
        S.interpolate_sparse(S.SparseField(v, m), np.zeros((6, 9), np.float32), S.SmoothConfig(r=0))
    assert str(e.value) == "smooth: r must be >= 1"


def test_sparse_errors_match_oracle(port):
    """Same texts as the CPU restatement for multi-fault inputs."""
    from oracle.pyoracle import OracleError

    cases = []
    v, m = _field(); m[2, 3] = 0.5; v[4, 4] = 1.0; cases.append((v, m, S.SmoothConfig()))
    v, m = _field(); m[0, 0] = 1.0; v[1, 1] = 2.0; cases.append((v, m, S.SmoothConfig(r=0)))
    v, m = _field(); cases.append((v, m, S.SmoothConfig(tau=9)))
    for v, m, cfg in cases:
        g = np.zeros(v.shape, np.float32)
        with pytest.raises(OracleError) as e1:
            port.interpolate_sparse(v, m, g, cfg)
        with pytest.raises(S.Error) as e2:
            S.interpolate_sparse(S.SparseField(v, m), g, cfg)
        assert str(e1.value) == str(e2.value)


def test_cabi_sparse_without_pixels_is_empty_mask():
    nc = N.to_native(S.SmoothConfig())
    err = N.errbuf()
    buf = np.zeros(4, np.float32)
    rc = N.lib().sgwls_b200_interpolate_sparse_batch(buf.ctypes.data, buf.ctypes.data, buf.ctypes.data, 1, 0, 4, 1,
                                                     1, C.byref(nc), buf.ctypes.data, None, err, len(err))
    assert rc == N.EINVAL
    assert err.value.decode() == "interpolate_sparse: empty mask"


def test_device_forms_reject_host_tensors():
    torch = pytest.importorskip("torch")
    t = torch.zeros((4, 4), dtype=torch.float32)
    with pytest.raises(S.Error, match="contiguous float32 CUDA tensor"):
        S.smooth_device(t, t)
    with pytest.raises(S.Error, match="contiguous float32 CUDA tensor"):
        S.interpolate_sparse_device(t[None], t[None], t[None])
