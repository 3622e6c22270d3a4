"""Compare the pass-0 super-separator values (SGWLS_DEBUG_Z dump) with exact band solves."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1705_01674_b200 as S
from oracle.pyoracle import CpuOracle
h, w, r, tau, NW = 200, 40, 1, 3, int(os.environ.get("SGWLS_TILE_WARPS", "8"))
rng = np.random.default_rng(0)
t = rng.uniform(0, 1, (h, w, 1)).astype(np.float32)
g = (np.round(rng.uniform(0, 1, (h, w, 1)) * 3) / 3).astype(np.float32)
cfg = S.SmoothConfig(lambda_=400.0, r=r, tau=tau, iterations=1, weight=S.WeightParams(kind=S.WeightKind.Exp, sigma_r=0.1))
os.environ["SGWLS_DEBUG_Z"] = "/tmp/z.bin"
S.smooth(t, g, cfg)
z = np.fromfile("/tmp/z.bin", dtype=np.float32)
orc = CpuOracle("port")
M = 2 * r + 1
RW = max(1, min(8, 64 // (M * (1 + r))))
P = (h + RW - 1) // RW
PS = (P + NW - 1) // NW
centers = orc.band_centers(w, r, tau)
nb = len(centers)
zz = z[: (PS - 1) * r * nb].reshape(PS - 1, r, nb)
worst = []
for b, cen in enumerate(centers):
    rows, cols = orc.band_layout(h, w, cen, r, 0)
    wts = orc.edge_weights(g[:, :, 0].astype(np.float64), cen, r, 0, cfg)
    rhs = t[rows, cols, 0].astype(np.float64)
    u, *_ = orc.solve_band(wts, 400.0, rhs, r)
    for J in range(PS - 1):
        lastrow = (J + 1) * NW * RW - 1
        for q in range(r):
            pos = lastrow * M + (M - r + q)
            worst.append((abs(zz[J, q, b] - u[pos]), J, b, q, float(zz[J, q, b]), float(u[pos])))
worst.sort(reverse=True)
print("RW", RW, "P", P, "PS", PS, "nb", nb)
print("worst separator errors:", worst[:6])
