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
outs = [S.smooth(t, g, cfg) for _ in range(5)]
print("runs identical:", all(np.array_equal(outs[0], o) for o in outs), " max err per run:", [float(np.abs(o - want).max()) for o in outs])
