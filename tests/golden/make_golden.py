"""Generate the golden fixtures from the REFERENCE library itself.

Run in the build container (where /root/reference exists and oracle/_ref is
built):  python tests/golden/make_golden.py
Writes tests/golden/golden.npz: seeded fp32 inputs, the configuration, and the
reference's double outputs of sgwls::smooth / sgwls::interpolate_sparse
(via oracle/_ref/libsgwls_ref.so, i.e. proj/src/smoother.cpp unmodified), plus
1-D band solves and band-centre lists.  The GPU box has no /root/reference;
these fixtures are what pins the C restatement there.
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle.pyoracle import CpuOracle  # noqa: E402
from paper_1705_01674_b200.config import Axis, SmoothConfig, WeightKind, WeightParams  # noqa: E402

# (h, w, c, cg, lambda, r, tau, T, kind, axis, sigma_r, gscale)
SMOOTH_CASES = [
    (17, 23, 1, 1, 400.0, 1, 1, 4, 1, 0, 0.1, 1.0),
    (12, 9, 3, 1, 900.0, 1, 3, 4, 0, 0, 3.0, 1.0),
    (9, 12, 3, 3, 300.0, 2, 2, 3, 1, 1, 0.2, 1.0),
    (1, 64, 1, 1, 50.0, 2, 1, 1, 1, 1, 0.1, 1.0),
    (64, 1, 1, 1, 50.0, 2, 1, 2, 1, 0, 0.1, 1.0),
    (5, 3, 1, 3, 300.0, 3, 4, 2, 0, 0, 3.0, 1.0),
    (2, 2, 1, 1, 300.0, 4, 9, 4, 1, 0, 0.1, 1.0),
    (1, 1, 1, 1, 300.0, 2, 3, 4, 1, 0, 0.1, 1.0),
    (31, 40, 1, 1, 900.0, 3, 2, 4, 1, 0, 0.05, 1.0),
    (40, 31, 3, 1, 100.0, 4, 4, 4, 1, 1, 3.0, 255.0),
    (25, 25, 1, 1, 0.0, 2, 2, 4, 1, 0, 0.1, 1.0),
    (33, 21, 1, 1, 900.0, 1, 1, 4, 0, 0, 3.0, 1.0),
]


def cfg_of(case):
    h, w, c, cg, lam, r, tau, T, kind, axis, sr, gs = case
    return SmoothConfig(lambda_=lam, r=r, tau=tau, iterations=T,
                        weight=WeightParams(kind=WeightKind(kind), sigma_r=sr, guidance_scale=gs),
                        first_axis=Axis(axis), threads=1)


def main():
    ref = CpuOracle("reference")
    rng = np.random.default_rng(20261019)
    out = {}
    meta = {"smooth": [], "sparse": [], "band": [], "centers": []}
    for i, case in enumerate(SMOOTH_CASES):
        h, w, c, cg = case[:4]
        t = rng.uniform(0, 1, (h, w, c)).astype(np.float32)
        g = (np.round(rng.uniform(0, 1, (h, w, cg)) * 4) / 4 + rng.normal(0, 0.03, (h, w, cg))).astype(np.float32)
        o = ref.smooth(t, g, cfg_of(case))
        out[f"smooth{i}_t"], out[f"smooth{i}_g"], out[f"smooth{i}_out"] = t, g, o
        meta["smooth"].append(list(case))
    for i, (h, w, r, tau) in enumerate([(30, 26, 2, 2), (17, 40, 1, 1)]):
        g = (np.round(rng.uniform(0, 1, (h, w)) * 3) / 3).astype(np.float32)
        m = (rng.uniform(0, 1, (h, w)) < 0.15).astype(np.float32)
        m[0, 0] = 1.0
        v = np.where(m > 0, rng.uniform(0.2, 1, (h, w)), 0).astype(np.float32)
        case = (h, w, 1, 1, 400.0, r, tau, 4, 1, 0, 0.05, 1.0)
        o, und = ref.interpolate_sparse(v, m, g, cfg_of(case))
        out[f"sparse{i}_v"], out[f"sparse{i}_m"], out[f"sparse{i}_g"] = v, m, g
        out[f"sparse{i}_out"], out[f"sparse{i}_und"] = o, und
        meta["sparse"].append(list(case))
    for i, (n, r, lam) in enumerate([(3, 1, 1.0), (57, 2, 400.0), (80, 3, 900.0), (40, 5, 10.0)]):
        wts = rng.uniform(0, 1, n * r)
        rhs = rng.uniform(0, 1, n)
        if i == 0:  # SPEC.md:179,197 tridiagonal example
            wts = np.array([1.0, 1.0, 0.0])
            rhs = np.array([1.0, 2.0, 3.0])
        u, alpha, beta, gamma = ref.solve_band(wts, lam, rhs, r)
        out[f"band{i}_w"], out[f"band{i}_rhs"] = wts, rhs
        out[f"band{i}_u"], out[f"band{i}_alpha"], out[f"band{i}_beta"], out[f"band{i}_gamma"] = u, alpha, beta, gamma
        meta["band"].append([n, r, lam])
    for ext, r, tau in [(9, 1, 1), (9, 1, 3), (10, 1, 4), (2048, 3, 2), (1080, 1, 3), (8192, 2, 3), (5, 3, 4),
                        (1, 2, 3), (7, 3, 7), (1920, 1, 3)]:
        meta["centers"].append([ext, r, tau, ref.band_centers(ext, r, tau)])
    out["meta"] = np.frombuffer(json.dumps(meta).encode(), dtype=np.uint8)
    np.savez_compressed(os.path.join(HERE, "golden.npz"), **out)
    print("wrote", os.path.join(HERE, "golden.npz"))


if __name__ == "__main__":
    main()
