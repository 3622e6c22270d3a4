"""The five BASELINE.json configurations and their seeded synthetic inputs.

The reference ships no dataset and no Voronoi generator (SURVEY.md §2
"Synthetic scenes"), so the inputs are generated here as SURVEY.md §8(d)
prescribes: uniform sites, each pixel centre (x+.5, y+.5) takes the nearest
site (ties -> lower site index, scipy cKDTree), U(0,1) cell values, then the
per-config texture / gradient / noise.  Seeds are ``1705 + 100*config + image``.

Parameter mapping: "range sigma" ->
WeightKind.Exp with sigma_r = sigma, guidance_scale = 1, sigma_s = 4 (reference
default), first_axis = Column; primary reading tau = the config's band stride
with iterations = 4; the secondary reading ("sweeps") is iterations = tau, tau = 1.
"""
from __future__ import annotations

import dataclasses

import numpy as np

from .config import Axis, SmoothConfig, WeightKind, WeightParams


@dataclasses.dataclass
class Workload:
    name: str
    width: int
    height: int
    channels: int          # target channels filtered per image
    batch: int             # images per filter call (c4: 64 pairs)
    sparse: bool           # interpolate_sparse (c4) instead of smooth
    cfg: SmoothConfig
    cells: int

    @property
    def pixels(self) -> int:
        return self.width * self.height * self.batch

    def bytes_alg(self) -> int:
        """Algorithmic HBM bytes per filter:
        B * [T * 4*M*N*(2C + G) + E], C = RHS channels per pass, G = 1 guidance
        channel, E = 4*M*N*3 for the sparse ratio epilogue."""
        m_n = self.width * self.height
        c = self.channels + (1 if self.sparse else 0)
        e = 4 * m_n * 3 if self.sparse else 0
        return self.batch * (self.cfg.iterations * 4 * m_n * (2 * c + 1) + e)


def _cfg(lam, r, tau, sigma, secondary=False) -> SmoothConfig:
    w = WeightParams(kind=WeightKind.Exp, sigma_s=4.0, sigma_r=sigma, guidance_scale=1.0)
    if secondary:
        return SmoothConfig(lambda_=lam, r=r, tau=1, iterations=tau, weight=w, first_axis=Axis.Column)
    return SmoothConfig(lambda_=lam, r=r, tau=tau, iterations=4, weight=w, first_axis=Axis.Column)


def workload(name: str, secondary: bool = False, batch: int | None = None) -> Workload:
    if name == "c1":
        w = Workload("c1", 512, 512, 1, 1, False, _cfg(400.0, 1, 1, 0.03, secondary), 64)
    elif name == "c2":
        w = Workload("c2", 1920, 1080, 3, 1, False, _cfg(400.0, 1, 3, 0.03, secondary), 256)
    elif name == "c3":
        w = Workload("c3", 2048, 2048, 1, 1, False, _cfg(900.0, 3, 2, 0.05, secondary), 512)
    elif name == "c4":
        w = Workload("c4", 1024, 1024, 1, 64, True, _cfg(400.0, 2, 2, 0.02, secondary), 128)
    elif name == "c5":
        w = Workload("c5", 8192, 8192, 1, 1, False, _cfg(400.0, 2, 3, 0.03, secondary), 4096)
    else:
        raise ValueError(f"unknown workload {name!r}")
    if batch is not None:
        w.batch = batch
    return w


# ----------------------------------------------------------------- generators

def voronoi_labels(width: int, height: int, cells: int, rng: np.random.Generator):
    """Nearest-site labels for pixel centres; returns (labels[h,w] int32, sites[cells,2] as (x,y))."""
    from scipy.spatial import cKDTree

    sites = rng.uniform(0.0, 1.0, size=(cells, 2)) * np.array([width, height])
    tree = cKDTree(sites)
    labels = np.empty((height, width), dtype=np.int32)
    xs = np.arange(width, dtype=np.float64) + 0.5
    step = max(1, (1 << 22) // width)
    for y0 in range(0, height, step):
        y1 = min(height, y0 + step)
        yy, xx = np.meshgrid(np.arange(y0, y1, dtype=np.float64) + 0.5, xs, indexing="ij")
        pts = np.stack([xx.ravel(), yy.ravel()], axis=1)
        _, idx = tree.query(pts, k=1, workers=-1)
        labels[y0:y1] = idx.reshape(y1 - y0, width)
    return labels, sites


def _seed(cfg_index: int, image: int) -> int:
    return 1705 + 100 * cfg_index + image


def gen_c1(image: int = 0, width=512, height=512):
    rng = np.random.default_rng(_seed(1, image))
    lab, _ = voronoi_labels(width, height, 64, rng)
    val = rng.uniform(0, 1, 64)[lab]
    img = np.clip(val + rng.normal(0, 0.05, lab.shape), 0, 1).astype(np.float32)
    return img, img


def gen_c2(image: int = 0, width=1920, height=1080):
    rng = np.random.default_rng(_seed(2, image))
    chans = []
    yy, xx = np.meshgrid(np.arange(height) + 0.5, np.arange(width) + 0.5, indexing="ij")
    for _c in range(3):
        lab, sites = voronoi_labels(width, height, 256, rng)
        base = rng.uniform(0, 1, 256)
        slope = rng.uniform(-0.2, 0.2, 256) / width
        theta = rng.uniform(0, 2 * np.pi, 256)
        dx = xx - sites[lab, 0]
        dy = yy - sites[lab, 1]
        ch = base[lab] + slope[lab] * (dx * np.cos(theta)[lab] + dy * np.sin(theta)[lab])
        ch = ch + rng.normal(0, 0.04, lab.shape)
        chans.append(np.clip(ch, 0, 1))
    rgb = np.stack(chans, axis=2).astype(np.float32)
    # BT.601 luma (proj/src/image.cpp:255,290-298), computed once in fp32
    luma = (np.float32(0.299) * rgb[:, :, 0] + np.float32(0.587) * rgb[:, :, 1]
            + np.float32(0.114) * rgb[:, :, 2]).astype(np.float32)
    return rgb, luma


def gen_c3(image: int = 0, width=2048, height=2048):
    rng = np.random.default_rng(_seed(3, image))
    lab, _ = voronoi_labels(width, height, 512, rng)
    base = rng.uniform(0, 1, 512)
    period = rng.uniform(4, 32, 512)
    theta = rng.uniform(0, 2 * np.pi, 512)
    phase = rng.uniform(0, 2 * np.pi, 512)
    yy, xx = np.meshgrid(np.arange(height) + 0.5, np.arange(width) + 0.5, indexing="ij")
    proj = xx * np.cos(theta)[lab] + yy * np.sin(theta)[lab]
    img = base[lab] + 0.05 * np.sin(2 * np.pi * proj / period[lab] + phase[lab])
    img = (img + rng.normal(0, 0.03, lab.shape)).astype(np.float32)
    return img, img


def gen_c4(image: int = 0, width=1024, height=1024):
    """One (values, mask, guidance) pair of the joint-filtering batch."""
    rng = np.random.default_rng(_seed(4, image))
    lab, sites = voronoi_labels(width, height, 128, rng)
    guide = rng.uniform(0, 1, 128)[lab].astype(np.float32)
    depth = rng.uniform(0.2, 1.0, 128)
    sx = rng.uniform(-1e-3, 1e-3, 128)
    sy = rng.uniform(-1e-3, 1e-3, 128)
    yy, xx = np.meshgrid(np.arange(height) + 0.5, np.arange(width) + 0.5, indexing="ij")
    plane = depth[lab] + sx[lab] * (xx - sites[lab, 0]) + sy[lab] * (yy - sites[lab, 1])
    mask = (rng.uniform(0, 1, lab.shape) < 1.0 / 16.0)
    vals = np.where(mask, plane + rng.normal(0, 0.01, lab.shape), 0.0).astype(np.float32)
    return vals, mask.astype(np.float32), guide


def gen_c5(image: int = 0, width=8192, height=8192):
    rng = np.random.default_rng(_seed(5, image))
    lab, _ = voronoi_labels(width, height, 4096, rng)
    img = (rng.uniform(0, 1, 4096)[lab] + rng.normal(0, 0.05, lab.shape)).astype(np.float32)
    return img, img


GENERATORS = {"c1": gen_c1, "c2": gen_c2, "c3": gen_c3, "c4": gen_c4, "c5": gen_c5}
