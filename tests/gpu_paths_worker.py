"""Subprocess body of tests/test_gpu_paths.py: parity of the tiled pass under
one forced kernel schedule (SGWLS_KA_WARPS / SGWLS_TILE_WARPS / SGWLS_K2_NG /
SGWLS_PDL are read once per process).  Prints the max |delta| per case."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1705_01674_b200 as S  # noqa: E402
from oracle.pyoracle import CpuOracle  # noqa: E402

CASES = [  # (h, w, c, r, tau, lam, T)
    (300, 257, 1, 1, 1, 900.0, 4),
    (270, 96, 3, 1, 3, 400.0, 2),
    (257, 300, 1, 2, 3, 400.0, 4),
    (200, 140, 2, 2, 2, 400.0, 3),
    (181, 99, 1, 3, 2, 900.0, 2),
    (140, 77, 1, 4, 5, 100.0, 2),
    (100, 68, 1, 1, 2, 400.0, 2),  # W, H multiples of 4, not of 32: vectorised transpose with edge tiles
    # shuffle averaging edge cases: a last tile of exactly 32 bands whose tail
    # columns have no writer lane (falls back to the phase path), a forced last
    # band centre off the tau grid, two channels
    (70, 64, 1, 1, 1, 900.0, 1),
    (90, 100, 1, 1, 2, 400.0, 2),
    (60, 100, 2, 2, 3, 400.0, 2),
    # rows on 16-byte bounds in both orientations (TMA-staged KB where the schedule allows),
    # several interior band tiles, r = 2 .. 4, a partial last row tile
    (328, 400, 1, 2, 3, 400.0, 4),
    (132, 260, 1, 2, 1, 300.0, 2),
    (184, 100, 1, 3, 2, 900.0, 2),
    (144, 80, 1, 4, 5, 100.0, 2),
    (96, 264, 3, 2, 2, 400.0, 2),
    # tall lines: long reduced systems
    (4100, 40, 2, 1, 2, 400.0, 2),
    (9000, 36, 1, 1, 1, 900.0, 1),
]
port = CpuOracle("port")
rng = np.random.default_rng(5)
worst = 0.0
for h, w, c, r, tau, lam, T in CASES:
    t = rng.random((h, w, c)).astype(np.float32)
    g = (np.round(rng.random((h, w)) * 4) / 4 + 0.02 * rng.standard_normal((h, w))).astype(np.float32)
    cfg = S.SmoothConfig(lambda_=lam, r=r, tau=tau, iterations=T,
                         weight=S.WeightParams(kind=S.WeightKind.Exp, sigma_r=0.1))
    d = float(np.abs(S.smooth(t, g, cfg) - port.smooth(t, g, cfg)).max())
    worst = max(worst, d)
    print(f"{h}x{w}x{c} r={r} tau={tau}: {d:.2e}")
print(f"WORST {worst:.3e}")
