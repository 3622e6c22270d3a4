import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1705_01674_b200 as S
from oracle.pyoracle import CpuOracle
h, w, c, r, tau, T, kind, axis = [int(a) for a in sys.argv[1:9]]
rng = np.random.default_rng(0)
t = rng.uniform(0, 1, (h, w, c)).astype(np.float32)
g = (np.round(rng.uniform(0, 1, (h, w, 1)) * 3) / 3).astype(np.float32)
cfg = S.SmoothConfig(lambda_=400.0, r=r, tau=tau, iterations=T, weight=S.WeightParams(kind=S.WeightKind(kind), sigma_r=0.1), first_axis=S.Axis(axis))
want = CpuOracle("port").smooth(t, g, cfg)
got = S.smooth(t, g, cfg)
np.set_printoptions(precision=4, linewidth=200, suppress=True)
for y in [34, 35, 36, 38, 40, 42, 44]:
    print(y, "got ", got[y, :12, 0])
    print(y, "want", want[y, :12, 0])
    print(y, "in  ", t[y, :12, 0])
