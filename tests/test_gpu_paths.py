"""Every kernel schedule of the tiled pass against the oracle: KA tile heights
(the tiles KA's separator maps span) independent of the KB tile heights, K2
tree widths, programmatic dependent launch on and off, KB's input staging (per-lane loads or
tensor-map TMA) and its lean interior body.  The schedule is chosen per radius by default, so each forced choice
runs in its own process (the knobs are read once)."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCHEDULES = [
    {"SGWLS_PDL": "1"},
    {"SGWLS_PDL": "0"},
    {"SGWLS_KA_WARPS": "4", "SGWLS_TILE_WARPS": "8"},
    {"SGWLS_KA_WARPS": "8", "SGWLS_TILE_WARPS": "2"},
    {"SGWLS_KA_WARPS": "3", "SGWLS_TILE_WARPS": "5", "SGWLS_K2_NG": "4"},
    {"SGWLS_KA_WARPS": "2", "SGWLS_K2_NG": "16"},
    {"SGWLS_KA_WARPS": "1"},
    # KB input staging: per-lane loads everywhere / tensor-map TMA for every r >= 2 (default: r = 2
    # only) / staged but without the lean interior body
    {"SGWLS_KB_STAGE": "0"},
    {"SGWLS_KB_STAGE": "1"},
    {"SGWLS_KB_LEAN": "0"},
    {"SGWLS_KB_STAGE": "1", "SGWLS_KA_WARPS": "4", "SGWLS_TILE_WARPS": "8", "SGWLS_PDL": "0"},
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
