"""Run one smooth() case on the GPU and report where it departs from the oracle."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1705_01674_b200 as S
from oracle.pyoracle import CpuOracle

def run(h, w, c, r, tau, T, kind, axis, lam=400.0, seed=0):
    rng = np.random.default_rng(seed)
    t = rng.uniform(0, 1, (h, w, c)).astype(np.float32)
    g = (np.round(rng.uniform(0, 1, (h, w, 1)) * 3) / 3).astype(np.float32)
    cfg = S.SmoothConfig(lambda_=lam, r=r, tau=tau, iterations=T,
                         weight=S.WeightParams(kind=S.WeightKind(kind), sigma_r=0.1), first_axis=S.Axis(axis))
    want = CpuOracle("port").smooth(t, g, cfg)
    got = S.smooth(t, g, cfg)
    d = np.abs(got - want)
    bad = ~(d <= 1e-4)
    print(f"{h}x{w}x{c} r={r} tau={tau} T={T} kind={kind} axis={axis}: max={np.nanmax(np.where(np.isnan(d), 0, d)):.3g} "
          f"nan={int(np.isnan(got).sum())} bad={int(bad.sum())}")
    if bad.any():
        ys, xs = np.nonzero(bad.any(axis=2))
        print("   bad rows", sorted(set(ys.tolist()))[:20], "cols", sorted(set(xs.tolist()))[:40])

CASES = [(40, 31, 3, 2, 2, 1, 0, 0), (40, 31, 3, 2, 2, 1, 0, 1), (40, 31, 1, 2, 2, 1, 1, 0), (64, 40, 1, 1, 1, 1, 1, 0),
             (64, 40, 1, 1, 3, 1, 1, 0), (64, 40, 3, 1, 3, 1, 1, 0), (64, 40, 1, 2, 5, 1, 1, 0), (64, 40, 1, 2, 3, 1, 1, 0),
             (200, 40, 1, 2, 5, 1, 1, 0), (200, 40, 1, 1, 3, 1, 1, 0), (200, 100, 1, 1, 1, 1, 1, 0),
             (200, 40, 1, 3, 7, 1, 1, 0), (512, 40, 1, 1, 3, 1, 1, 0)]
if __name__ == "__main__":
    for args in CASES:
        run(*args)
