"""Time the multi-GPU C ABI (sgwls_b200_smooth_multi) with G slabs on device 0
against the single-device host call, on c5 (host buffers in and out, like e2e).
usage: python scripts/multi_local.py [G ...]"""
import ctypes as C
import json
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_1705_01674_b200 as S  # noqa: E402
from paper_1705_01674_b200 import _native as N  # noqa: E402
from paper_1705_01674_b200 import workloads as WL  # noqa: E402

wl = WL.workload("c5")
t, g = WL.GENERATORS["c5"](0)
cfg = wl.cfg
out = np.empty_like(t)
nc = N.to_native(cfg)
err = N.errbuf()
res = {}
for G in [1] + [int(x) for x in sys.argv[1:]]:
    devs = np.zeros(G, np.int32)

    def call():
        rc = N.lib().sgwls_b200_smooth_multi(t.ctypes.data, wl.width, wl.height, 1, g.ctypes.data, 1, C.byref(nc),
                                             devs.ctypes.data, G, out.ctypes.data, err, len(err))
        N.check(rc, err)

    call()
    ref = out.copy() if G == 1 else ref
    t0 = time.perf_counter()
    n = 5
    for _ in range(n):
        call()
    el = (time.perf_counter() - t0) / n
    res[G] = {"ms": el * 1e3, "max_diff_vs_G1": float(np.abs(out - ref).max())}
    print(G, res[G], flush=True)
print(json.dumps(res))
