"""Line-slab sharded filter (paper_1705_01674_b200/sharded.py).

CPU: the window algebra is checked with the oracle as the per-pass compute --
sharded (in one process, and over a world_size-2 gloo group) must be
BIT-identical to the same pass sequence unsharded.  GPU: the native pass
through the same orchestration against smooth_device and the oracle.
"""
import os
import socket

import numpy as np
import pytest

from paper_1705_01674_b200.config import Axis, SmoothConfig, WeightKind, WeightParams
from paper_1705_01674_b200.sharded import LocalExchange, ShardedSmoother, plan_windows


def _cfg(r=2, tau=3, T=4, lam=400.0, sr=0.05, fa=Axis.Column):
    return SmoothConfig(lambda_=lam, r=r, tau=tau, iterations=T, first_axis=fa,
                        weight=WeightParams(kind=WeightKind.Exp, sigma_r=sr))


def _img(h, w, c=1, seed=0):
    rng = np.random.default_rng(seed)
    base = rng.random((h // 8 + 1, w // 8 + 1, c)).repeat(8, 0).repeat(8, 1)[:h, :w]
    return np.clip(base + 0.05 * rng.standard_normal((h, w, c)), 0, 1).astype(np.float32)


def oracle_pass(port):
    """Per-pass compute for the CPU tests: one Column pass of the C oracle, transposed, fp32."""
    import torch

    def run(src, guid, cfg, out):
        res = port.smooth(src.numpy(), guid.numpy(), cfg)  # (Hl, wl, C) float64
        out.copy_(torch.from_numpy(res.astype(np.float32)).transpose(0, 1))
        return out
    return run


def unsharded_passes(port, t, g, cfg):
    """The same pass sequence on one shard (fp32 between passes, like the sharded pipeline)."""
    sm = ShardedSmoother(t.shape[0], t.shape[1], t.shape[2], g.shape[2], cfg, exchange=LocalExchange(1),
                         device="cpu", pass_fn=oracle_pass(port))
    sm.load(t, g)
    sm.run()
    return sm.gather().numpy()


@pytest.mark.parametrize("extent,G,r,tau", [(100, 2, 1, 1), (100, 3, 2, 3), (64, 4, 3, 2), (57, 5, 2, 5),
                                             (41, 2, 4, 9), (8192, 8, 2, 3)])
def test_plan_windows_cover_exact_bands(extent, G, r, tau, port):
    wins = plan_windows(extent, G, r, tau)
    assert wins[0].oa == 0 and wins[-1].ob == extent
    glob = set(port.band_centers(extent, r, tau))
    for a, b in zip(wins, wins[1:]):
        assert a.ob == b.oa
    for w in wins:
        assert w.s % tau == 0 and 0 <= w.s <= w.oa < w.ob <= w.e <= extent
        loc = [c + w.s for c in port.band_centers(w.width, r, tau)]
        # every band touching an owned column is a global band, and every global band doing so is local
        touch_loc = {c for c in loc if c + r >= w.oa and c - r < w.ob}
        touch_glob = {c for c in glob if c + r >= w.oa and c - r < w.ob}
        assert touch_loc == touch_glob


@pytest.mark.parametrize("G,cfg,shape", [
    (2, _cfg(r=1, tau=1, T=2), (40, 52, 1)),
    (3, _cfg(r=2, tau=3, T=4), (45, 61, 1)),
    (4, _cfg(r=3, tau=2, T=3, lam=900.0), (70, 66, 2)),
    (2, _cfg(r=2, tau=5, T=4, fa=Axis.Row), (33, 48, 3)),
])
def test_local_shards_bit_identical(G, cfg, shape, port):
    h, w, c = shape
    t = _img(h, w, c, seed=G)
    g = _img(h, w, 1, seed=100 + G)
    ref = unsharded_passes(port, t, g, cfg)
    sm = ShardedSmoother(h, w, c, 1, cfg, exchange=LocalExchange(G), device="cpu", pass_fn=oracle_pass(port))
    sm.load(t, g)
    sm.run()
    out = sm.gather().numpy()
    assert out.shape == (h, w, c)
    assert np.array_equal(out, ref)
    # and the fp32-between-passes pipeline stays within the parity bar of the reference smooth
    full = port.smooth(t, g, cfg)
    assert np.abs(out - full).max() < 1e-5


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _gloo_worker(rank, world, port_no, q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port_no)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle.pyoracle import CpuOracle
        from paper_1705_01674_b200.sharded import DistExchange

        port = CpuOracle("port")
        cfg = _cfg(r=2, tau=3, T=4)
        t = _img(50, 47, 1, seed=7)
        g = _img(50, 47, 1, seed=8)
        sm = ShardedSmoother(50, 47, 1, 1, cfg, exchange=DistExchange(), device="cpu", pass_fn=oracle_pass(port))
        sm.load(t, g)
        sm.run()
        a, b, own = sm.owned()
        full = sm.gather().numpy()
        ref = unsharded_passes(port, t, g, cfg)
        q.put((rank, a, b, bool(np.array_equal(full, ref)), float(np.abs(full - ref).max())))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_bit_identical():
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port_no = _free_port()
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port_no, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert [r[0] for r in res] == [0, 1]
    assert res[0][1] == 0 and res[0][2] == res[1][1]  # owned ranges tile the extent
    assert all(r[3] for r in res), res


@pytest.mark.gpu
@pytest.mark.parametrize("G,cfg,shape", [
    (3, _cfg(r=2, tau=3, T=4), (300, 257, 1)),
    (2, _cfg(r=1, tau=3, T=4, lam=400.0, sr=0.03), (270, 480, 3)),
    (4, _cfg(r=3, tau=2, T=3, lam=900.0), (512, 200, 1)),
])
def test_gpu_local_shards_match_unsharded(G, cfg, shape, port):
    import torch

    import paper_1705_01674_b200 as S

    h, w, c = shape
    t = _img(h, w, c, seed=G)
    g = _img(h, w, 1, seed=10 + G)
    sm = ShardedSmoother(h, w, c, 1, cfg, exchange=LocalExchange(G), device="cuda")
    sm.load(t, g)
    sm.run()
    out = sm.gather().cpu().numpy()
    dev = S.smooth_device(torch.from_numpy(t).cuda(), torch.from_numpy(g).cuda(), cfg, sync=True).cpu().numpy()
    ref = port.smooth(t, g, cfg)
    d_dev = float(np.abs(out - dev).max())
    d_ref = float(np.abs(out - ref).max())
    print(f"sharded G={G}: max|d| vs unsharded GPU {d_dev:.2e}, vs oracle {d_ref:.2e}")
    assert d_dev < 2e-6
    assert d_ref < 1e-4
