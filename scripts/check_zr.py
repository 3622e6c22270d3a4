import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1705_01674_b200 as S
from oracle.pyoracle import CpuOracle
h, w, r, tau = 200, 40, 1, 3
rng = np.random.default_rng(0)
t = rng.uniform(0, 1, (h, w, 1)).astype(np.float32)
g = (np.round(rng.uniform(0, 1, (h, w, 1)) * 3) / 3).astype(np.float32)
cfg = S.SmoothConfig(lambda_=400.0, r=r, tau=tau, iterations=1, weight=S.WeightParams(kind=S.WeightKind.Exp, sigma_r=0.1))
os.environ["SGWLS_DEBUG_ZR"] = "/tmp/zr.bin"
got = S.smooth(t, g, cfg)
orc = CpuOracle("port")
want = orc.smooth(t, g, cfg)
print("max err", float(np.abs(got - want).max()))
M = 3; RW = 8; P = 25
centers = orc.band_centers(w, r, tau); nb = len(centers)
d = np.fromfile("/tmp/zr.bin", dtype=np.float32).reshape(P, 2, nb)
for b, cen in enumerate(centers[:5]):
    rows, cols = orc.band_layout(h, w, cen, r, 0)
    wts = orc.edge_weights(g[:, :, 0].astype(np.float64), cen, r, 0, cfg)
    u, *_ = orc.solve_band(wts, 400.0, t[rows, cols, 0].astype(np.float64), r)
    bad = []
    for j in range(P):
        if j < P - 1:
            pos = (j + 1) * RW * M - 1
            if abs(d[j, 1, b] - u[pos]) > 1e-5: bad.append(("zr", j, float(d[j, 1, b]), float(u[pos])))
        if j > 0:
            pos = j * RW * M - 1
            if abs(d[j, 0, b] - u[pos]) > 1e-5: bad.append(("zl", j, float(d[j, 0, b]), float(u[pos])))
    print("band", b, bad[:6])
