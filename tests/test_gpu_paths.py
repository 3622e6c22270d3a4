"""Every kernel schedule of the tiled pass against the oracle: KB solving its
tile's inner separators vs the separate KC launch, KA/KB tile heights, K2 fused
into KA, KB waiting on per-band-group ready flags, both grid orders.  The schedule is chosen per radius by default, so each forced choice
runs in its own process (the knobs are read once)."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCHEDULES = [
    {"SGWLS_KC": "0"},
    {"SGWLS_KC": "1"},
    {"SGWLS_KC": "1", "SGWLS_KA_WARPS": "4", "SGWLS_TILE_WARPS": "8"},
    {"SGWLS_KC": "0", "SGWLS_TILE_WARPS": "2"},
    {"SGWLS_KC": "0", "SGWLS_FUSE_K2": "1"},
    {"SGWLS_KC": "0", "SGWLS_FLAGS": "1"},
    {"SGWLS_KC": "0", "SGWLS_FLAGS": "1", "SGWLS_KA_JFAST": "1", "SGWLS_KB_JFAST": "1"},
    {"SGWLS_KC": "1", "SGWLS_FUSE_K2": "1", "SGWLS_KA_WARPS": "2"},
]


@pytest.mark.gpu
@pytest.mark.parametrize("env", SCHEDULES, ids=lambda e: ",".join(f"{k[6:]}={v}" for k, v in e.items()))
def test_schedule_parity(env):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "gpu_paths_worker.py")], cwd=ROOT,
                       env={**os.environ, **env}, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    worst = float(r.stdout.strip().splitlines()[-1].split()[-1])
    print(env, f"worst {worst:.2e}")
    assert worst <= 1e-4, r.stdout
