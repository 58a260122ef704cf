"""Seeded synthetic workloads of BASELINE.json's five configs (setup only, never timed).

No public dataset is involved: every config is a seeded piecewise-constant phantom blurred by a
parametric PSF plus Gaussian noise at an exact level. What BASELINE leaves open is
fixed here and recorded in DESIGN.md:

* phantom: shapes painted in order with overwrite onto a zero image — first all rectangles
  (side lengths uniform integers in [max(2, m//64), max(3, m//8)]), then all disks (radius uniform
  in [max(1, m/128), max(2, m/16)]); intensities U[0,1]; RNG ``np.random.default_rng(seed)``.
* PSFs: sampled on an odd w x w grid centred at ((w+1)/2, (w+1)/2), clipped to >= 0 and
  normalised to sum 1 (psf.py:56); ``pad_to`` then fixes the band anchor.
* data: b = exact blur of the phantom (blur_direct semantics, psf.py:170-193) + Gaussian noise
  rescaled to level*||b|| (imaging.py:141-167, Philox substream "noise").
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .errors import ArgumentError
from .psf import BoundaryCondition, Psf
from .rand import stream


@dataclass(frozen=True)
class Config:
    name: str
    m: int
    batch: int
    dtypes: tuple
    bc: str
    w: int
    r: int
    lam: float
    iters: int
    noise: float
    n_rect: int
    n_disk: int
    psf: str


CONFIGS = {
    "cfg1": Config("cfg1", 256, 1, ("float64",), "zero", 31, 3, 0.02, 100, 0.01, 40, 20, "gauss_rot"),
    "cfg2": Config("cfg2", 1024, 1, ("float64", "float32"), "reflective", 63, 5, 0.01, 200, 0.005, 200, 100, "two_gauss"),
    "cfg3": Config("cfg3", 512, 512, ("float32",), "zero", 31, 4, 0.02, 100, 0.01, 100, 50, "gauss_random"),
    "cfg4": Config("cfg4", 4096, 1, ("float32",), "zero", 255, 8, 0.005, 300, 0.01, 2000, 1000, "moffat"),
    "cfg5": Config("cfg5", 16384, 1, ("float32",), "reflective", 127, 10, 0.01, 100, 0.01, 20000, 10000, "motion"),
}


# ------------------------------------------------------------------------------ phantoms
def phantom_shapes(m: int, n_rect: int, n_disk: int, seed: int):
    rng = np.random.default_rng(seed)
    lo, hi = max(2, m // 64), max(3, m // 8)
    rects = []
    for _ in range(n_rect):
        h = int(rng.integers(lo, hi + 1))
        w = int(rng.integers(lo, hi + 1))
        r0 = int(rng.integers(0, max(1, m - h + 1)))
        c0 = int(rng.integers(0, max(1, m - w + 1)))
        rects.append((r0, c0, h, w, float(rng.random())))
    rlo, rhi = max(1.0, m / 128), max(2.0, m / 16)
    disks = []
    for _ in range(n_disk):
        rad = float(rng.uniform(rlo, rhi))
        ci = float(rng.uniform(0, m - 1))
        cj = float(rng.uniform(0, m - 1))
        disks.append((ci, cj, rad, float(rng.random())))
    return rects, disks


def phantom(m: int, n_rect: int, n_disk: int, seed: int, device="cpu"):
    """Piecewise-constant phantom as a float64 torch tensor (painting is exact assignment, so
    the result is identical on any device)."""
    import torch

    rects, disks = phantom_shapes(m, n_rect, n_disk, seed)
    X = torch.zeros((m, m), dtype=torch.float64, device=device)
    for r0, c0, h, w, v in rects:
        X[r0 : r0 + h, c0 : c0 + w] = v
    for ci, cj, rad, v in disks:
        i0, i1 = max(0, int(math.floor(ci - rad))), min(m, int(math.ceil(ci + rad)) + 1)
        j0, j1 = max(0, int(math.floor(cj - rad))), min(m, int(math.ceil(cj + rad)) + 1)
        ii = torch.arange(i0, i1, device=device, dtype=torch.float64)[:, None] - ci
        jj = torch.arange(j0, j1, device=device, dtype=torch.float64)[None, :] - cj
        mask = ii * ii + jj * jj <= rad * rad
        sub = X[i0:i1, j0:j1]
        sub[mask] = v
    return X


# ------------------------------------------------------------------------------ PSFs
def _grid(w: int):
    c = (w - 1) / 2.0
    d = np.arange(w) - c
    return d[:, None], d[None, :]  # (row offset, col offset)


def _rot_gauss(w: int, s_major: float, s_minor: float, angle: float) -> np.ndarray:
    y, x = _grid(w)
    ca, sa = math.cos(angle), math.sin(angle)
    u = ca * x + sa * y
    v = -sa * x + ca * y
    g = np.exp(-0.5 * ((u / s_major) ** 2 + (v / s_minor) ** 2))
    return g / g.sum()


def _moffat(w: int, core: float, beta: float) -> np.ndarray:
    y, x = _grid(w)
    g = (1.0 + (x * x + y * y) / core**2) ** (-beta)
    return g / g.sum()


def _motion(w: int, length: float, angle: float, sigma: float) -> np.ndarray:
    """Bilinearly deposited line of `length` px at `angle`, convolved with a Gaussian."""
    line = np.zeros((w, w))
    c = (w - 1) / 2.0
    steps = int(math.ceil(length)) * 8 + 1
    for t in np.linspace(-(length - 1) / 2.0, (length - 1) / 2.0, steps):
        x = c + t * math.cos(angle)
        y = c - t * math.sin(angle)
        x0, y0 = int(math.floor(x)), int(math.floor(y))
        fx, fy = x - x0, y - y0
        for dy, wy in ((0, 1 - fy), (1, fy)):
            for dx, wx in ((0, 1 - fx), (1, fx)):
                if 0 <= y0 + dy < w and 0 <= x0 + dx < w:
                    line[y0 + dy, x0 + dx] += wy * wx
    yy, xx = _grid(w)
    h = int(math.ceil(4 * sigma))
    k = np.exp(-0.5 * (np.arange(-h, h + 1) / sigma) ** 2)
    k /= k.sum()
    out = np.apply_along_axis(lambda r: np.convolve(r, k, mode="same"), 1, line)
    out = np.apply_along_axis(lambda r: np.convolve(r, k, mode="same"), 0, out)
    out = np.maximum(out, 0.0)
    return out / out.sum()


def make_psf(cfg: Config, index: int = 0, seed: int = 0) -> Psf:
    w = cfg.w
    if cfg.psf == "gauss_rot":
        v = _rot_gauss(w, 4.0, 1.5, math.radians(30.0))
    elif cfg.psf == "two_gauss":
        v = 0.7 * _rot_gauss(w, 6.0, 2.0, math.radians(15.0)) + 0.3 * _rot_gauss(w, 3.0, 3.0, 0.0)
    elif cfg.psf == "gauss_random":
        rng = np.random.default_rng([seed, index, 7])
        v = _rot_gauss(w, float(rng.uniform(2, 5)), float(rng.uniform(1, 2)), float(rng.uniform(0, math.pi)))
    elif cfg.psf == "moffat":
        v = _moffat(w, 12.0, 2.5)
    elif cfg.psf == "motion":
        v = _motion(w, 41.0, math.radians(15.0), 2.0)
    else:  # pragma: no cover
        raise ArgumentError(f"unknown psf family {cfg.psf}")
    v = np.maximum(v, 0.0)
    v = v / v.sum()
    c = (w + 1) // 2
    return Psf(v, (c, c))


# ------------------------------------------------------------------------------ data
def blur_exact(X, psf: Psf, bc: str):
    """blur_direct (psf.py:170-193) for a torch float64 image. On the GPU this is the native
    kb_blur_direct kernel (bit-identical to the reference); CPU tensors (CPU-only tests of this
    harness) take symmetric / zero padding plus a torch conv2d correlation with the flipped PSF."""
    import torch
    import torch.nn.functional as F

    if X.is_cuda:
        from .blur import blur_direct

        return blur_direct(psf, X, bc)

    rows, cols = psf.values.shape
    l, q = psf.center
    m, n = X.shape
    top, bot, lef, rig = rows - l, l - 1, cols - q, q - 1
    if bc == "zero":
        Xp = F.pad(X[None, None], (lef, rig, top, bot))[0, 0]
    else:  # numpy "symmetric": edge sample repeated, single reflection (rows <= m)
        ri = torch.arange(-top, m + bot, device=X.device)
        ci = torch.arange(-lef, n + rig, device=X.device)
        ri = torch.where(ri < 0, -1 - ri, torch.where(ri >= m, 2 * m - 1 - ri, ri))
        ci = torch.where(ci < 0, -1 - ci, torch.where(ci >= n, 2 * n - 1 - ci, ci))
        Xp = X[ri][:, ci]
    P = torch.as_tensor(np.ascontiguousarray(psf.values[::-1, ::-1]), dtype=torch.float64, device=X.device)
    return F.conv2d(Xp[None, None], P[None, None])[0, 0]


def add_noise(b: np.ndarray, level: float, seed: int) -> np.ndarray:
    """Gaussian noise with ||noise|| = level * ||b|| exactly (imaging.py:141-167, kind "gauss")."""
    b = np.asarray(b, dtype=float)
    norm_b = float(np.linalg.norm(b.ravel()))
    if norm_b == 0:
        raise ArgumentError("cannot scale noise against zero data")
    if level == 0:
        return b.copy()
    for attempt in range(8):
        g = stream(seed, "noise", index=attempt).standard_normal(b.shape)
        norm_g = float(np.linalg.norm(g.ravel()))
        if norm_g > 0:
            return b + (level * norm_b / norm_g) * g
    raise ArgumentError("noise draw degenerated")  # pragma: no cover


def make_image_data(cfg: Config, seed: int = 0, index: int = 0, device="cpu", m: int | None = None,
                    counts: tuple | None = None):
    """(truth X, psf, noisy data B) for one image of a config, float64 numpy arrays.

    ``m`` / ``counts`` override the size and shape counts (smaller parity cases of a config)."""
    m = cfg.m if m is None else int(m)
    nr, nd = (cfg.n_rect, cfg.n_disk) if counts is None else counts
    X = phantom(m, nr, nd, seed * 100003 + index, device=device)
    psf = make_psf(cfg, index=index, seed=seed)
    b = blur_exact(X, psf, cfg.bc).cpu().numpy()
    B = add_noise(b, cfg.noise, seed * 100003 + index)
    return X.cpu().numpy(), psf, B
