"""Row-slab sharded filter: one image across G GPUs with the band solves
partitioned exactly across the GPUs -- no image transposes
between GPUs.

Every GPU keeps a fixed slab of image rows [a, b) (a even: the serpentine
parity of proj/src/snake.cpp:21-49 stays the local one) for the whole filter.

* Column passes (bands run down the rows, across every slab): the partitioned
  solve of sgwls_tile.cuh "row-slab mode".  Phase A (``sgwls_b200_slab_pass_a``)
  computes the slab's chunk records and ONE record per band for the whole slab;
  the G slab records per band (~100 B each, ~0.1-0.3 MB per GPU for 8192^2)
  are all-gathered; phase B (``sgwls_b200_slab_pass_b``) solves the G-1 slab
  separators of every band (the same tiny block-tridiagonal system on every
  GPU), then the slab's own separators and chunk interiors, and writes the
  slab's rows.  Exact: the same elimination as the single-GPU pass, regrouped.
* Row passes (bands run along rows, each 2r+1 rows tall): a row band only
  reads its own rows, so each GPU computes the bands covering its rows on a
  row window [s, e) ⊇ [a, b) (``sharded.plan_windows`` algebra), after a halo
  exchange of the <= 2r+1 neighbouring rows on each side, then keeps rows
  [a, b).  The window is transposed on the device and run as an ordinary
  Column pass (``pass_device``), whose output is written transposed back.

Per pass transition a GPU therefore sends O(r * W) floats of halo rows and
O(G * bands) floats of slab records, instead of the (G-1)/G^2 of the image
that the all-to-all transpose of ``sharded.ShardedSmoother`` moves.

``LocalExchange`` runs all slabs in one process (validation on one device);
``DistExchange`` one slab per rank (NCCL; gloo for the host-logic tests).
"""
from __future__ import annotations

import ctypes as C

from . import _native as N
from .config import Axis, Error, SmoothConfig
from .sharded import DistExchange, LocalExchange, Window  # noqa: F401  (re-exported)


def slab_rows(height: int, nslabs: int) -> list[tuple[int, int]]:
    """Balanced slabs [a, b) with even starts (serpentine parity)."""
    if nslabs < 1:
        raise Error("sharded: need at least one shard")
    bounds = [2 * ((g * height) // (2 * nslabs)) for g in range(nslabs)] + [height]
    out = [(bounds[g], bounds[g + 1]) for g in range(nslabs)]
    if any(b <= a for a, b in out):
        raise Error(f"sharded: height {height} is too small for {nslabs} row slabs")
    return out


def row_windows(height: int, slabs: list[tuple[int, int]], r: int, tau: int) -> list[Window]:
    """Window [s, e) of the row pass around each slab (same algebra as sharded.plan_windows)."""
    out = []
    for oa, ob in slabs:
        s = 0 if oa == 0 else (max(0, oa - 2 * r) // tau) * tau
        e = height if ob == height else min(height, ob + 2 * r + 1)
        out.append(Window(s, e, oa, ob))
    return out


def _transpose(src, dst) -> None:
    """(H, W, C) -> (W, H, C) with the library's transpose kernel."""
    import torch

    h, w, c = src.shape
    err = N.errbuf()
    with torch.cuda.device(src.device):
        st = torch.cuda.current_stream(src.device).cuda_stream
        N.check(N.lib().sgwls_b200_transpose_device(src.data_ptr(), dst.data_ptr(), 1, w, h, c, C.c_void_p(st), err,
                                                    len(err)), err)


class SlabSmoother:
    """``sgwls::smooth`` (proj/src/smoother.cpp:113-125) of ONE image over G row slabs.

    ``load(target, guidance)`` keeps this process's slab (+ windows) resident on
    ``device``; ``run()`` performs the T passes; ``owned()`` / ``gather()``
    return the result rows."""

    def __init__(self, height: int, width: int, channels: int, guidance_channels: int, cfg: SmoothConfig,
                 exchange=None, device=None):
        import torch

        from .api import validate

        validate(cfg)
        self.H, self.W, self.C, self.Cg = height, width, channels, guidance_channels
        self.cfg = cfg
        self.ex = exchange if exchange is not None else DistExchange()
        self.G = self.ex.nshards
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.pcfg = cfg.copy(iterations=1, first_axis=Axis.Column)
        self.slabs = slab_rows(height, self.G)
        self.win = row_windows(height, self.slabs, cfg.r, cfg.tau)
        self.T = cfg.iterations
        self.fa = int(Axis(cfg.first_axis))
        self.nc = N.to_native(self.pcfg)
        self._alloc()

    def _sizes(self, rows: int):
        work, rec = C.c_size_t(), C.c_size_t()
        err = N.errbuf()
        N.check(N.lib().sgwls_b200_slab_sizes(self.W, rows, self.C, self.Cg, self.G, C.byref(self.nc), C.byref(work),
                                              C.byref(rec), err, len(err)), err)
        return work.value, rec.value

    def _alloc(self) -> None:
        import torch

        dev, W, Cc, Cg = self.device, self.W, self.C, self.Cg
        f32 = dict(dtype=torch.float32, device=dev)
        self.buf, self.gwin, self.gwinT, self.tmpT, self.work = {}, {}, {}, {}, {}
        recn = None
        for g in self.ex.local:
            a, b = self.slabs[g]
            w = self.win[g]
            self.buf[g] = [torch.empty((w.width, W, Cc), **f32) for _ in range(2)]  # ping-pong row windows
            self.gwin[g] = torch.empty((w.width, W, Cg), **f32)  # guidance rows [s, e)
            self.gwinT[g] = torch.empty((W, w.width, Cg), **f32)
            self.tmpT[g] = torch.empty((W, w.width, Cc), **f32)
            work, recn = self._sizes(b - a)
            self.work[g] = torch.empty(max(work, 1), **f32)
        self.recn = recn
        self.allrec = {g: torch.empty((self.G, recn), **f32) for g in self.ex.local}
        # first-pass pivot-failure word per local slab (sgwls_b200_slab_pass_b)
        self.errw = {g: torch.full((1,), -1, dtype=torch.int64, device=dev) for g in self.ex.local}

    @staticmethod
    def _hwc(a):
        import numpy as np
        import torch

        t = torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)) if isinstance(a, np.ndarray) else a
        if t.dim() == 2:
            t = t.unsqueeze(-1)
        return t

    def load(self, target, guidance) -> None:
        t = self._hwc(target)
        gd = self._hwc(guidance)
        if tuple(t.shape) != (self.H, self.W, self.C) or tuple(gd.shape) != (self.H, self.W, self.Cg):
            raise Error("smooth: target and guidance dimensions differ")
        for g in self.ex.local:
            a, b = self.slabs[g]
            w = self.win[g]
            self.buf[g][0][a - w.s:b - w.s].copy_(t[a:b])
            self.gwin[g].copy_(gd[w.s:w.e])
            _transpose(self.gwin[g], self.gwinT[g])
        self.cur = 0

    def _guid_rows(self, g: int):
        """Guidance from slab row a on; row a-1 (the previous slab's last) precedes it in memory."""
        return self.gwin[g][self.slabs[g][0] - self.win[g].s:]

    def host_windows(self, target, guidance) -> dict:
        """This process's slab rows and guidance window as pinned host tensors (for load_windows)."""
        import torch

        t = self._hwc(target)
        gd = self._hwc(guidance)
        pin = (lambda x: x.contiguous().pin_memory()) if torch.cuda.is_available() else (lambda x: x.contiguous())
        out = {}
        for g in self.ex.local:
            a, b = self.slabs[g]
            w = self.win[g]
            out[g] = (pin(t[a:b]), pin(gd[w.s:w.e]))
        return out

    def load_windows(self, windows: dict) -> None:
        """Stream-ordered upload of host_windows() output (slab rows + guidance window)."""
        for g, (x, gw) in windows.items():
            self._own(g, 0).copy_(x, non_blocking=True)
            self.gwin[g].copy_(gw, non_blocking=True)
            _transpose(self.gwin[g], self.gwinT[g])
        self.cur = 0

    def window_bytes(self) -> int:
        return sum(4 * (self._own(g, 0).numel() + self.gwin[g].numel()) for g in self.ex.local)

    def kernel_launches(self) -> int:
        """Native kernels one run() launches in this process."""
        from .api import kernel_launches

        n = 0
        for p in range(self.T):
            for g in self.ex.local:
                if ((self.fa + p) & 1) == 0:  # KA, slab reduce | slab solve, KB
                    n += 4
                else:  # window transpose + one pass
                    n += 1 + kernel_launches(self.win[g].width, self.W, self.C, self.Cg, 1, False, self.pcfg)
        return n

    # ---------------------------------------------------------------- passes
    def _own(self, g: int, k: int):
        a, b = self.slabs[g]
        s = self.win[g].s
        return self.buf[g][k][a - s:b - s]

    def _column_pass(self, first: bool = False) -> None:
        nxt = self.cur ^ 1
        err = N.errbuf()
        for g in self.ex.local:
            a, b = self.slabs[g]
            src = self._own(g, self.cur)
            guid = self._guid_rows(g)
            st = C.c_void_p(self._stream(g))
            N.check(N.lib().sgwls_b200_slab_pass_a(src.data_ptr(), guid.data_ptr(), self.W, b - a, self.C, self.Cg,
                                                   a, self.G, g, C.byref(self.nc), self.work[g].data_ptr(),
                                                   self.allrec[g][g].data_ptr(), st, err, len(err)), err)
        self._gather_records()
        for g in self.ex.local:
            a, b = self.slabs[g]
            src = self._own(g, self.cur)
            guid = self._guid_rows(g)
            out = self._own(g, nxt)
            st = C.c_void_p(self._stream(g))
            ew = self.errw[g].data_ptr() if first else None
            N.check(N.lib().sgwls_b200_slab_pass_b(src.data_ptr(), guid.data_ptr(), self.W, b - a, self.C, self.Cg,
                                                   a, self.G, g, C.byref(self.nc), self.work[g].data_ptr(),
                                                   self.allrec[g].data_ptr(), out.data_ptr(), ew, st, err,
                                                   len(err)), err)
        self.cur = nxt

    def _row_pass(self, first: bool = False) -> None:
        from .api import pass_device

        self._halo_exchange()
        nxt = self.cur ^ 1
        for g in self.ex.local:
            _transpose(self.buf[g][self.cur], self.tmpT[g])
            # Column pass on the transposed window, written transposed: rows [s, e) of the image.
            # A first (row) pass synchronises to report the reference's pivot failure.
            pass_device(self.tmpT[g], self.gwinT[g], self.pcfg, out=self.buf[g][nxt], graph=True, sync=first)
        self.cur = nxt

    def _stream(self, g: int) -> int:
        import torch

        return torch.cuda.current_stream(self.device).cuda_stream

    def _gather_records(self) -> None:
        """allrec[g][h] = slab h's record, for every local g (all-gather)."""
        sends, recvs = [], []
        for g in self.ex.local:
            for h in range(self.G):
                if h == g:
                    continue
                if h in self.ex.local:
                    self.allrec[h][g].copy_(self.allrec[g][g])
                else:
                    sends.append((h, self.allrec[g][g]))
                    recvs.append((h, self.allrec[g][h]))
        self.ex.run(sends, recvs)

    def _halo_exchange(self) -> None:
        """Rows of the window [s, e) outside the slab come from the slabs that own them."""
        k = self.cur
        sends, recvs = [], []
        for g in self.ex.local:
            a, b = self.slabs[g]
            for h in range(self.G):
                if h == g:
                    continue
                wh = self.win[h]
                lo, hi = max(a, wh.s), min(b, wh.e)  # my rows inside h's window
                if lo < hi:
                    src = self.buf[g][k][lo - self.win[g].s:hi - self.win[g].s]
                    if h in self.ex.local:
                        self.buf[h][k][lo - wh.s:hi - wh.s].copy_(src)
                    else:
                        sends.append((h, src))
                ah, bh = self.slabs[h]
                lo, hi = max(ah, self.win[g].s), min(bh, self.win[g].e)  # h's rows inside my window
                if lo < hi and h not in self.ex.local:
                    recvs.append((h, self.buf[g][k][lo - self.win[g].s:hi - self.win[g].s]))
        self.ex.run(sends, recvs)

    def close(self) -> None:
        """Release the CUDA graphs this smoother's passes captured (process-wide graph cache)."""
        from .api import graph_clear

        graph_clear()

    def run(self) -> None:
        import torch

        # the native calls launch on the current device: make it this smoother's
        with torch.cuda.device(self.device):
            for g in self.ex.local:
                self.errw[g].fill_(-1)
            for p in range(self.T):
                if ((self.fa + p) & 1) == 0:
                    self._column_pass(first=p == 0)
                else:
                    self._row_pass(first=p == 0)

    def check_errors(self) -> None:
        """Raise the reference's pivot failure (proj/src/banded.cpp:66-68) if the
        first pass met one on any slab: the smallest (line, position) key wins,
        as in the unsharded filter.  Synchronises (and, distributed, gathers the
        keys of all ranks)."""
        keys = [int(self.errw[g].item()) & 0xFFFFFFFFFFFFFFFF for g in self.ex.local]
        if len(self.ex.local) < self.G:
            keys = self.ex.all_gather_int(min(keys))
        key = min(keys)
        if key != 0xFFFFFFFFFFFFFFFF:
            raise Error(f"rband_lu_factorize: non-positive pivot at row {key & 0xFFFFFFFF} (input not SPD)")

    def owned(self, g: int | None = None):
        """(first, last, rows): slab g's rows [first, last) of the result (H-major layout)."""
        g = self.ex.local[0] if g is None else g
        a, b = self.slabs[g]
        return a, b, self._own(g, self.cur)

    def gather(self):
        """Full (H, W, C) result on every process (raises the first pass's pivot failure)."""
        import torch

        self.check_errors()
        full = torch.empty((self.H, self.W, self.C), dtype=torch.float32, device=self.device)
        for g in self.ex.local:
            a, b, t = self.owned(g)
            full[a:b].copy_(t)
        if len(self.ex.local) < self.G:
            for g in range(self.G):
                a, b = self.slabs[g]
                part = full[a:b].contiguous()
                self.ex.broadcast(part, g)
                full[a:b].copy_(part)
        return full


def smooth_slabs(target, guidance, cfg: SmoothConfig | None = None, exchange=None, device=None):
    """One-shot ``smooth`` of one image over row slabs; returns the full (H, W[, C])."""
    cfg = cfg or SmoothConfig()
    t = SlabSmoother._hwc(target)
    gd = SlabSmoother._hwc(guidance)
    H, W, Cc = t.shape
    sm = SlabSmoother(H, W, Cc, gd.shape[2], cfg, exchange=exchange, device=device)
    sm.load(t, gd)
    sm.run()
    out = sm.gather()
    return out if getattr(target, "ndim", 3) == 3 else out[:, :, 0]
