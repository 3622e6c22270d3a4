"""Row-slab sharded filter with the band solves partitioned across GPUs
(paper_1705_01674_b200/slabs.py, sgwls_tile.cuh row-slab mode).

CPU: the slab / window algebra, and the two exchanges (slab-record all-gather,
halo rows) over a world_size-2 gloo group on CPU tensors.  GPU: G slabs in one
process on one device (LocalExchange) against the unsharded filter and the
oracle, for every kernel schedule (r = 1 in-KB separators, r >= 2 KC), both
first axes, T = 1..4, one and three channels, slabs down to a single chunk.
"""
import os
import socket

import numpy as np
import pytest

from paper_1705_01674_b200.config import Axis, SmoothConfig, WeightKind, WeightParams
from paper_1705_01674_b200.slabs import LocalExchange, SlabSmoother, row_windows, slab_rows


def _cfg(r=2, tau=3, T=4, lam=400.0, sr=0.05, fa=Axis.Column):
    return SmoothConfig(lambda_=lam, r=r, tau=tau, iterations=T, first_axis=fa,
                        weight=WeightParams(kind=WeightKind.Exp, sigma_r=sr))


def _img(h, w, c=1, seed=0):
    rng = np.random.default_rng(seed)
    base = rng.random((h // 8 + 1, w // 8 + 1, c)).repeat(8, 0).repeat(8, 1)[:h, :w]
    return np.clip(base + 0.05 * rng.standard_normal((h, w, c)), 0, 1).astype(np.float32)


@pytest.mark.parametrize("H,G,r,tau", [(100, 2, 1, 1), (101, 3, 2, 3), (64, 4, 3, 2), (57, 5, 2, 5), (8192, 8, 2, 3)])
def test_slab_rows_and_windows(H, G, r, tau, port):
    slabs = slab_rows(H, G)
    assert slabs[0][0] == 0 and slabs[-1][1] == H
    for (a, b), (c, d) in zip(slabs, slabs[1:]):
        assert b == c
    assert all(a % 2 == 0 and b > a for a, b in slabs)
    glob = set(port.band_centers(H, r, tau))
    for w in row_windows(H, slabs, r, tau):
        assert w.s % tau == 0 and 0 <= w.s <= w.oa < w.ob <= w.e <= H
        loc = {c + w.s for c in port.band_centers(w.width, r, tau)}
        need = {c for c in glob if c + r >= w.oa and c - r < w.ob}  # global bands touching owned rows
        assert need <= loc and {c for c in loc if c + r >= w.oa and c - r < w.ob} <= glob


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _gloo_worker(rank, world, port_no, q):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port_no)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1705_01674_b200.slabs import DistExchange

        H, W = 40, 23
        cfg = _cfg(r=2, tau=3, T=2)
        sm = SlabSmoother(H, W, 1, 1, cfg, exchange=DistExchange(), device="cpu")
        a, b = sm.slabs[rank]
        w = sm.win[rank]
        # rows carry their global index: after the halo exchange the whole window must
        for k in (0, 1):
            sm.buf[rank][k].fill_(-1.0)
        own = torch.arange(a, b, dtype=torch.float32)[:, None, None].expand(b - a, W, 1)
        sm.buf[rank][0][a - w.s:b - w.s].copy_(own)
        sm.cur = 0
        sm._halo_exchange()
        rows = sm.buf[rank][0][:, 0, 0]
        halo_ok = bool(torch.equal(rows, torch.arange(w.s, w.e, dtype=torch.float32)))
        sm.allrec[rank][rank].fill_(float(rank + 1))
        sm._gather_records()
        rec_ok = all(bool(torch.all(sm.allrec[rank][h] == h + 1)) for h in range(world))
        q.put((rank, halo_ok, rec_ok))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_exchanges():
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
    assert res == [(0, True, True), (1, True, True)], res


@pytest.mark.gpu
@pytest.mark.parametrize("G,cfg,shape", [
    (2, _cfg(r=2, tau=3, T=4), (300, 257, 1)),
    (3, _cfg(r=2, tau=3, T=4), (301, 130, 1)),
    (4, _cfg(r=1, tau=3, T=4, lam=400.0, sr=0.03), (270, 480, 3)),
    (3, _cfg(r=1, tau=1, T=2, lam=900.0), (200, 96, 1)),
    (4, _cfg(r=3, tau=2, T=3, lam=900.0), (512, 200, 1)),
    (2, _cfg(r=4, tau=5, T=1, lam=100.0), (160, 90, 2)),
    (3, _cfg(r=2, tau=2, T=4, fa=Axis.Row), (150, 170, 1)),
    (8, _cfg(r=2, tau=3, T=2), (64, 140, 1)),   # 8-row slabs: two chunks each
    (8, _cfg(r=2, tau=3, T=4), (24, 140, 1)),   # 2-4-row slabs: one chunk each, windows span several slabs
    (1, _cfg(r=2, tau=3, T=4), (120, 100, 1)),
])
def test_gpu_slabs_match_unsharded(G, cfg, shape, port):
    import torch

    import paper_1705_01674_b200 as S

    h, w, c = shape
    t = _img(h, w, c, seed=G)
    g = _img(h, w, 1, seed=10 + G)
    sm = SlabSmoother(h, w, c, 1, cfg, exchange=LocalExchange(G), device="cuda")
    sm.load(t, g)
    sm.run()
    out = sm.gather().cpu().numpy()
    dev = S.smooth_device(torch.from_numpy(t).cuda(), torch.from_numpy(g).cuda(), cfg, sync=True).cpu().numpy()
    ref = port.smooth(t, g, cfg)
    d_dev = float(np.abs(out - dev).max())
    d_ref = float(np.abs(out - ref).max())
    print(f"slabs G={G} {shape} r={cfg.r}: max|d| vs unsharded GPU {d_dev:.2e}, vs oracle {d_ref:.2e}")
    assert d_ref < 1e-4
    assert d_dev < 2e-6


@pytest.mark.gpu
@pytest.mark.parametrize("fa", [Axis.Column, Axis.Row])
def test_gpu_slabs_report_pivot_failure(fa, port):
    """A NaN guidance sample is the reference's "non-positive pivot at row k"
    (proj/src/banded.cpp:66-68): the slab filter reports the same text."""
    import paper_1705_01674_b200 as S
    from oracle.pyoracle import OracleError

    h, w = 120, 90
    t = _img(h, w, 1, seed=4)
    g = _img(h, w, 1, seed=5)
    g[77, 41, 0] = np.nan  # in the third of three slabs
    cfg = _cfg(r=2, tau=3, T=2, fa=fa)
    with pytest.raises(OracleError) as want:
        port.smooth(t, g, cfg)
    sm = SlabSmoother(h, w, 1, 1, cfg, exchange=LocalExchange(3), device="cuda")
    sm.load(t, g)
    with pytest.raises(S.Error) as got:
        sm.run()
        sm.gather()
    assert str(got.value) == str(want.value)


def _gloo_gpu_worker(rank, world, port_no, q):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port_no)
    torch.cuda.set_device(0)  # both ranks share the one GPU; gloo stages through host memory
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1705_01674_b200.slabs import DistExchange

        h, w = 301, 130
        cfg = _cfg(r=2, tau=3, T=4)
        t = _img(h, w, 1, seed=21)
        g = _img(h, w, 1, seed=22)
        sm = SlabSmoother(h, w, 1, 1, cfg, exchange=DistExchange(), device="cuda:0")
        sm.load(t, g)
        sm.run()
        out = sm.gather().cpu().numpy()
        sm.close()
        if rank == 0:
            np.save(os.environ["SGWLS_TEST_OUT"], out)
        q.put((rank, "ok"))
    except Exception as e:  # reported to the parent
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
def test_gpu_slabs_two_processes_dist_exchange(port, tmp_path):
    """Two ranks (torch.distributed, gloo, both on cuda:0 -- the multi-rank code
    path with real process boundaries) run a full T = 4 slab filter; the
    gathered image matches the oracle."""
    import torch.multiprocessing as mp

    outp = str(tmp_path / "slab2.npy")
    os.environ["SGWLS_TEST_OUT"] = outp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port_no = _free_port()
    procs = [ctx.Process(target=_gloo_gpu_worker, args=(r, 2, port_no, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=600) for _ in procs)
    for p in procs:
        p.join(timeout=120)
    assert res == [(0, "ok"), (1, "ok")], res
    h, w = 301, 130
    t = _img(h, w, 1, seed=21)
    g = _img(h, w, 1, seed=22)
    want = port.smooth(t, g, _cfg(r=2, tau=3, T=4))
    got = np.load(outp)
    err = float(np.abs(got - want).max())
    print(f"2-process slab filter vs oracle: {err:.2e}")
    assert err <= 1e-4
