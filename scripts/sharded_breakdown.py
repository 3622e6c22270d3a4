"""Stage timing of the sharded pipeline on one GPU (LocalExchange): passes vs transposes."""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_1705_01674_b200 import workloads as WL  # noqa: E402
from paper_1705_01674_b200.sharded import LocalExchange, ShardedSmoother  # noqa: E402

wl = WL.workload("c5")
ht, hg = WL.GENERATORS["c5"](0)
for G in (1, 2, 4):
    sm = ShardedSmoother(wl.height, wl.width, 1, 1, wl.cfg, exchange=LocalExchange(G))
    sm.load(ht, hg)
    for _ in range(3):
        sm.run()
    torch.cuda.synchronize()
    ev = {}
    lay = 0
    tp = tx = 0.0
    for rep in range(5):
        for p in range(sm.T):
            lay = sm.layout(p)
            a, b, c = (torch.cuda.Event(enable_timing=True) for _ in range(3))
            a.record()
            for g in sm.ex.local:
                sm.pass_fn(sm.cur[g, lay], sm.guid[g, lay], sm.pcfg, sm.tmp[g, lay])
            b.record()
            if p + 1 < sm.T:
                sm._transpose_exchange(lay)
            c.record()
            torch.cuda.synchronize()
            tp += a.elapsed_time(b)
            tx += b.elapsed_time(c)
    print(f"G={G}: passes {tp / 5:.3f} ms/filter, transposes {tx / 5:.3f} ms/filter")
