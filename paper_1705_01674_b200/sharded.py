"""Line-slab sharded filter: one image across several GPUs (BASELINE c5).

The reference runs a pass as independent bands (``run_pass``,
proj/src/smoother.cpp:51-99) over an extent split into band centres
(``band_centers``, proj/src/snake.cpp:7-19).  A band only reads its own
2r+1 columns, and a column's average only involves the bands whose window
covers it.  So one pass shards exactly over column WINDOWS:

* shard g OWNS output columns [oa, ob) of the pass extent;
* it runs the ordinary single-device pass on the sub-image of columns
  [s, e) where s = the largest multiple of tau <= oa - 2r (then every local
  centre r + k*tau is a global centre) and e = ob + 2r + 1 (the window's own
  forced last centre, proj/src/snake.cpp:15-17, stays clear of the owned
  columns) -- both clamped to the image, where the window then coincides with
  the global geometry;
* every band covering an owned column is then a band of the window, computed
  from the same inputs, and averaged in the same centre order, so the owned
  columns equal the unsharded pass (bit-identical for the CPU oracle).

Every pass writes its output transposed (sgwls_b200_pass_device), so a shard
ends a pass holding complete ROWS [oa, ob) of the next layout, while the next
pass needs column windows of it.  Between passes the shards therefore do one
all-to-all transpose: shard g sends rows [oa_g, ob_g) x window columns of
shard h to h, which lands contiguously at rows [oa_g, ob_g) of h's next
window (NCCL grouped send/recv; NCCL has no alltoallv).  The guidance is fixed
across passes (proj/src/smoother.cpp:121): each shard keeps its windows of it
in both layouts, cut once at load time.

Shards either live one per process (``DistExchange`` over a
torch.distributed group: NCCL on GPUs, gloo for the CPU tests) or all in one
process (``LocalExchange``: validation of the window algebra on one device).
The per-pass compute is pluggable: the product path is the native
``pass_device``; the CPU tests plug the oracle in.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, Sequence

from .config import Axis, Error, SmoothConfig


@dataclass(frozen=True)
class Window:
    """Shard geometry along one pass extent (global column indices)."""
    s: int   # first window column
    e: int   # one past the last window column
    oa: int  # first owned column
    ob: int  # one past the last owned column

    @property
    def width(self) -> int:
        return self.e - self.s


def plan_windows(extent: int, nshards: int, r: int, tau: int) -> list[Window]:
    """Owned ranges (balanced, contiguous) and the exact-pass windows around them."""
    if nshards < 1:
        raise Error("sharded: need at least one shard")
    if nshards == 1 or extent < 2 * r + 1:
        if nshards != 1:
            raise Error(f"sharded: extent {extent} is too small for {nshards} shards at r={r}")
        return [Window(0, extent, 0, extent)]
    out = []
    for g in range(nshards):
        oa = g * extent // nshards
        ob = (g + 1) * extent // nshards
        if ob <= oa:
            raise Error(f"sharded: extent {extent} is too small for {nshards} shards")
        s = 0 if oa == 0 else (max(0, oa - 2 * r) // tau) * tau
        e = extent if ob == extent else min(extent, ob + 2 * r + 1)
        out.append(Window(s, e, oa, ob))
    return out


# ------------------------------------------------------------------ exchange

class LocalExchange:
    """All shards in this process; blocks move by copy."""

    def __init__(self, nshards: int):
        self.nshards = nshards
        self.local = list(range(nshards))

    def run(self, sends, recvs) -> None:  # pragma: no cover - no remote peers
        if sends or recvs:
            raise RuntimeError("LocalExchange has no remote peers")


class DistExchange:
    """One shard per rank of a torch.distributed group (NCCL or gloo)."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.nshards = dist.get_world_size(group)
        self.local = [dist.get_rank(group)]

    def _global(self, peer: int) -> int:
        return self.dist.get_global_rank(self.group, peer) if self.group is not None else peer

    def _staged(self, t) -> bool:
        # gloo moves host memory: device tensors travel through host copies
        return t.is_cuda and self.dist.get_backend(self.group) != "nccl"

    def run(self, sends, recvs) -> None:
        """sends/recvs: lists of (peer, tensor); one grouped exchange."""
        dist = self.dist
        if not sends and not recvs:
            return
        backend = dist.get_backend(self.group)
        if backend == "nccl":
            ops = [dist.P2POp(dist.isend, t, self._global(p), self.group) for p, t in sends]
            ops += [dist.P2POp(dist.irecv, t, self._global(p), self.group) for p, t in recvs]
            for w in dist.batch_isend_irecv(ops):
                w.wait()
            return
        # gloo: plain isend/irecv pairs on host tensors
        hs = [(p, t.contiguous().cpu() if self._staged(t) else t) for p, t in sends]
        hr = [(p, t, t.new_empty(t.shape, device="cpu") if self._staged(t) else t) for p, t in recvs]
        works = [dist.isend(h, self._global(p), self.group) for p, h in hs]
        works += [dist.irecv(h, self._global(p), self.group) for p, _, h in hr]
        for w in works:
            w.wait()
        for _, t, h in hr:
            if h is not t:
                t.copy_(h)

    def broadcast(self, t, src: int) -> None:
        """t (contiguous) from shard ``src`` to every shard, in place."""
        if self._staged(t):
            h = t.cpu()
            self.dist.broadcast(h, src=self._global(src), group=self.group)
            t.copy_(h)
        else:
            self.dist.broadcast(t, src=self._global(src), group=self.group)

    def all_gather_int(self, v: int) -> list:
        """Python ints (64-bit) of every shard."""
        import torch

        dev = "cuda" if self.dist.get_backend(self.group) == "nccl" else "cpu"
        x = torch.tensor([v - (1 << 64) if v >= (1 << 63) else v], dtype=torch.int64, device=dev)
        out = [torch.empty_like(x) for _ in range(self.nshards)]
        self.dist.all_gather(out, x, group=self.group)
        return [int(o.item()) & 0xFFFFFFFFFFFFFFFF for o in out]


# ------------------------------------------------------------------ passes

def native_pass(src, guid, cfg: SmoothConfig, out, graph: bool = True):
    """Product pass: sgwls_b200_pass_device (one Column pass, transposed output), graph-replayed."""
    from .api import pass_device

    return pass_device(src, guid, cfg, out=out, graph=graph)


class ShardedSmoother:
    """``sgwls::smooth`` (proj/src/smoother.cpp:113-125) of ONE image, line-slab sharded.

    ``load(target, guidance)`` cuts this process's windows out of the full
    (H, W[, C]) arrays (numpy or torch, any device) and keeps them resident on
    ``device``; ``run()`` performs the T passes with the all-to-all transposes
    between them, device-resident; ``owned()`` returns the rows of the result
    this process owns; ``gather()`` assembles the full result on every process.
    """

    def __init__(self, height: int, width: int, channels: int, guidance_channels: int, cfg: SmoothConfig,
                 exchange=None, device=None, pass_fn: Callable | None = None):
        import torch

        from .api import validate

        validate(cfg)
        self.H, self.W, self.C, self.Cg = height, width, channels, guidance_channels
        self.cfg = cfg
        self.ex = exchange if exchange is not None else DistExchange()
        self.G = self.ex.nshards
        self.device = torch.device(device) if device is not None else (
            torch.device("cuda", torch.cuda.current_device()) if torch.cuda.is_available() else torch.device("cpu"))
        self.pass_fn = pass_fn or native_pass
        self.pcfg = cfg.copy(iterations=1, first_axis=Axis.Column)
        # layout 0 = the image (bands across W, lines along H); layout 1 = its transpose
        self.ext = (width, height)        # pass extent (columns) per layout
        self.line = (height, width)       # line length (rows) per layout
        self.win = (plan_windows(width, self.G, cfg.r, cfg.tau), plan_windows(height, self.G, cfg.r, cfg.tau))
        self.T = cfg.iterations
        self.fa = int(Axis(cfg.first_axis))
        self._alloc()

    # layout of pass p
    def layout(self, p: int) -> int:
        return (self.fa + p) & 1

    def _alloc(self) -> None:
        import torch

        dev, C, Cg = self.device, self.C, self.Cg
        self.cur, self.guid, self.tmp = {}, {}, {}
        for g in self.ex.local:
            for lay in (0, 1):
                w = self.win[lay][g]
                self.cur[g, lay] = torch.empty((self.line[lay], w.width, C), dtype=torch.float32, device=dev)
                self.guid[g, lay] = torch.empty((self.line[lay], w.width, Cg), dtype=torch.float32, device=dev)
                self.tmp[g, lay] = torch.empty((w.width, self.line[lay], C), dtype=torch.float32, device=dev)
        self.sendbuf = {}
        for g in self.ex.local:
            for lay in (0, 1):
                w = self.win[lay][g]
                for h in range(self.G):
                    if h in self.ex.local:
                        continue
                    wn = self.win[1 - lay][h]
                    self.sendbuf[g, lay, h] = torch.empty((w.ob - w.oa, wn.width, C), dtype=torch.float32,
                                                          device=dev)

    @staticmethod
    def _hwc(a):
        import numpy as np
        import torch

        t = torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)) if isinstance(a, np.ndarray) else a
        if t.dim() == 2:
            t = t.unsqueeze(-1)
        return t

    def load(self, target, guidance) -> None:
        """Cut this process's windows (both layouts of the guidance, the first pass's layout of the target)."""
        t = self._hwc(target)
        gd = self._hwc(guidance)
        if tuple(t.shape) != (self.H, self.W, self.C) or tuple(gd.shape) != (self.H, self.W, self.Cg):
            raise Error("smooth: target and guidance dimensions differ")
        lay0 = self.layout(0)
        for g in self.ex.local:
            w0, w1 = self.win[0][g], self.win[1][g]
            self.guid[g, 0].copy_(gd[:, w0.s:w0.e, :])
            self.guid[g, 1].copy_(gd.transpose(0, 1)[:, w1.s:w1.e, :])
            src = t if lay0 == 0 else t.transpose(0, 1)
            w = self.win[lay0][g]
            self.cur[g, lay0].copy_(src[:, w.s:w.e, :])

    def host_windows(self, target, guidance) -> dict:
        """This process's input windows as pinned host tensors (for load_windows)."""
        import torch

        t = self._hwc(target)
        gd = self._hwc(guidance)
        lay0 = self.layout(0)
        src = t if lay0 == 0 else t.transpose(0, 1)
        out = {}
        for g in self.ex.local:
            w0, w1, w = self.win[0][g], self.win[1][g], self.win[lay0][g]
            out[g] = tuple(x.contiguous().pin_memory() if torch.cuda.is_available() else x.contiguous() for x in (
                src[:, w.s:w.e, :], gd[:, w0.s:w0.e, :], gd.transpose(0, 1)[:, w1.s:w1.e, :]))
        return out

    def load_windows(self, windows: dict) -> None:
        """Stream-ordered (non-blocking) upload of host_windows() output."""
        lay0 = self.layout(0)
        for g, (tw, g0, g1) in windows.items():
            self.cur[g, lay0].copy_(tw, non_blocking=True)
            self.guid[g, 0].copy_(g0, non_blocking=True)
            self.guid[g, 1].copy_(g1, non_blocking=True)

    def window_bytes(self) -> int:
        """Input bytes one load_windows() moves for this process."""
        lay0 = self.layout(0)
        return sum(4 * (self.cur[g, lay0].numel() + self.guid[g, 0].numel() + self.guid[g, 1].numel())
                   for g in self.ex.local)

    def kernel_launches(self) -> int:
        """Native kernels one run() launches in this process."""
        from .api import kernel_launches

        n = 0
        for p in range(self.T):
            lay = self.layout(p)
            for g in self.ex.local:
                n += kernel_launches(self.win[lay][g].width, self.line[lay], self.C, self.Cg, 1, False, self.pcfg)
        return n

    def _owned_rows(self, g: int, lay: int):
        """Rows [oa, ob) of the transposed pass output of shard g (a view of tmp)."""
        w = self.win[lay][g]
        return self.tmp[g, lay][w.oa - w.s:w.ob - w.s]

    def close(self) -> None:
        """Release the CUDA graphs this smoother's passes captured (process-wide graph cache)."""
        from .api import graph_clear

        graph_clear()

    def run(self) -> None:
        import contextlib

        import torch

        # the native calls launch on the current device: make it this smoother's
        ctx = torch.cuda.device(self.device) if self.device.type == "cuda" else contextlib.nullcontext()
        with ctx:
            for p in range(self.T):
                lay = self.layout(p)
                for g in self.ex.local:
                    self.pass_fn(self.cur[g, lay], self.guid[g, lay], self.pcfg, self.tmp[g, lay])
                if p + 1 < self.T:
                    self._transpose_exchange(lay)

    def _transpose_exchange(self, lay: int) -> None:
        nxt = 1 - lay
        sends, recvs = [], []
        for g in self.ex.local:
            own = self._owned_rows(g, lay)
            wg = self.win[lay][g]
            for h in range(self.G):
                wh = self.win[nxt][h]
                block = own[:, wh.s:wh.e, :]
                if h in self.ex.local:
                    self.cur[h, nxt][wg.oa:wg.ob].copy_(block)
                else:
                    buf = self.sendbuf[g, lay, h]
                    buf.copy_(block)
                    sends.append((h, buf))
        for h in self.ex.local:
            wh = self.win[nxt][h]
            for g in range(self.G):
                if g in self.ex.local:
                    continue
                wg = self.win[lay][g]
                recvs.append((g, self.cur[h, nxt][wg.oa:wg.ob]))
        self.ex.run(sends, recvs)

    def final_layout(self) -> int:
        """Layout of the result rows: 0 -> rows of the image, 1 -> columns of the image."""
        return 1 - self.layout(self.T - 1)

    def owned(self, g: int | None = None):
        """(first, last, tensor): shard g's rows [first, last) of the result in final_layout()."""
        g = self.ex.local[0] if g is None else g
        lay = self.layout(self.T - 1)
        w = self.win[lay][g]
        return w.oa, w.ob, self._owned_rows(g, lay)

    def gather(self):
        """Full (H, W, C) result on every process (torch tensor on self.device)."""
        import torch

        lay = self.layout(self.T - 1)
        full = torch.empty((self.ext[lay], self.line[lay], self.C), dtype=torch.float32, device=self.device)
        for g in self.ex.local:
            a, b, t = self.owned(g)
            full[a:b].copy_(t)
        if len(self.ex.local) < self.G:
            import torch.distributed as dist

            parts = [full[self.win[lay][g].oa:self.win[lay][g].ob].contiguous() for g in range(self.G)]
            for g in range(self.G):
                dist.broadcast(parts[g], src=self.ex._global(g), group=self.ex.group)
                w = self.win[lay][g]
                full[w.oa:w.ob].copy_(parts[g])
        return full if self.final_layout() == 0 else full.transpose(0, 1).contiguous()


def smooth_sharded(target, guidance, cfg: SmoothConfig | None = None, exchange=None, device=None,
                   pass_fn: Callable | None = None):
    """One-shot ``smooth`` of one image sharded over the exchange's shards; returns the full (H, W[, C])."""
    cfg = cfg or SmoothConfig()
    t = ShardedSmoother._hwc(target)
    gd = ShardedSmoother._hwc(guidance)
    H, W, C = t.shape
    sm = ShardedSmoother(H, W, C, gd.shape[2], cfg, exchange=exchange, device=device, pass_fn=pass_fn)
    sm.load(t, gd)
    sm.run()
    out = sm.gather()
    return out if getattr(target, "ndim", 3) == 3 else out[:, :, 0]


__all__: Sequence[str] = ["Window", "plan_windows", "LocalExchange", "DistExchange", "ShardedSmoother",
                          "smooth_sharded", "native_pass"]
