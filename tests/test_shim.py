"""The C++ drop-in shim (paper_1705_01674_b200/csrc/shim/smoother_gpu.cpp)
replaces proj/src/smoother.cpp under the reference's own application code
(proj/src/apps.cpp).  oracle/_ref/apps_ref links the reference smoother,
oracle/_ref/apps_gpu links the shim + libsgwls_b200.so, oracle/_ref/apps_gpu_dev
also replaces proj/src/apps.cpp with the device-pipeline shim (shim/apps_gpu.cpp);
all run the same pipelines (tests/cpp/apps_main.cpp) and must agree."""
import os
import subprocess
import tempfile

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_BIN = os.path.join(ROOT, "oracle", "_ref", "apps_ref")
GPU_BIN = os.path.join(ROOT, "oracle", "_ref", "apps_gpu")
DEV_BIN = os.path.join(ROOT, "oracle", "_ref", "apps_gpu_dev")

TOL = {"detail_enhance": 5e-4, "tone_map": 2e-3, "depth_upsample": 1e-4, "colorize": 1e-3}


def _run(binary):
    d = tempfile.mkdtemp()
    r = subprocess.run([binary, d], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    outs = {}
    for name in TOL:
        raw = open(os.path.join(d, name + ".bin"), "rb").read()
        w, h, c = np.frombuffer(raw[:12], dtype=np.int32)
        outs[name] = np.frombuffer(raw[12:], dtype=np.float64).reshape(h, w, c)
    return outs, r.stdout


@pytest.mark.gpu
@pytest.mark.parametrize("binary", [GPU_BIN, DEV_BIN], ids=["smoother_shim", "smoother_and_apps_shims"])
def test_reference_apps_on_gpu_shim(binary):
    if not (os.path.exists(REF_BIN) and os.path.exists(binary)):
        pytest.skip("apps binaries not built (needs /root/reference at build time)")
    ref, ref_out = _run(REF_BIN)
    gpu, gpu_out = _run(binary)
    assert gpu_out == ref_out  # identical sgwls::Error text on the invalid config
    for name, tol in TOL.items():
        a, b = gpu[name], ref[name]
        scale = max(1.0, float(np.abs(b).max()))
        err = float(np.abs(a - b).max()) / scale
        print(f"{name}: max rel-to-range |d| = {err:.3g}")
        assert err <= tol, name


@pytest.mark.parametrize("binary", [GPU_BIN, DEV_BIN], ids=["smoother_shim", "smoother_and_apps_shims"])
def test_apps_binaries_link_the_product_library(binary):
    if not os.path.exists(binary):
        pytest.skip("apps binaries not built")
    out = subprocess.run(["ldd", binary], capture_output=True, text=True).stdout
    assert "libsgwls_b200.so" in out
