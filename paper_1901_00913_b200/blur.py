"""Exact blur on the GPU: kronblur's ``blur_direct`` (psf.py:170-193) through ``kb_blur_direct``.

The reference pads the image (zero or numpy "symmetric" mode) and sums, for every nonzero PSF
entry in row-major order, the entry times a shifted slice of the padded image. The kernel replays
that per-pixel sequence with the same separately rounded fp64 products and sums
(``csrc/kb_blur.cuh``), so its output is bit-identical to the reference. It is used as the data
generator for the large configs (hours on the CPU at 4096² / 16384²) and as
the ``exact_apply`` callable of the history metrics (solvers.py:182, pipeline.py:180,294).

All-zero PSF borders are cropped on the host first (they add nothing; the centre moves with the
crop, so every remaining product reads the same image sample).
"""

from __future__ import annotations

import numpy as np

from .device import KB_BC_REFLECTIVE, KB_BC_ZERO, _check, _ptr, _stream_handle, _torch, load_library
from .errors import ArgumentError
from .psf import bc_name


def _crop(values: np.ndarray, center) -> tuple[np.ndarray, int, int]:
    """Smallest block holding every nonzero of `values` ([..., rows, cols]) and the centre in it."""
    nz = np.asarray(values != 0.0)
    if nz.ndim == 3:
        nz = nz.any(axis=0)
    rows = np.flatnonzero(nz.any(axis=1))
    cols = np.flatnonzero(nz.any(axis=0))
    l, q = int(center[0]), int(center[1])
    if rows.size == 0:  # unreachable for a valid Psf (sum 1); keep one entry
        return values[..., :1, :1], 1, 1
    r0, r1, c0, c1 = int(rows[0]), int(rows[-1]) + 1, int(cols[0]), int(cols[-1]) + 1
    return values[..., r0:r1, c0:c1], l - r0, q - c0


def _launch(psf_values: np.ndarray, center, X, bc, per_image: bool):
    """X: CUDA float64 tensor (batch, m, n), contiguous. Returns a new tensor."""
    torch = _torch()
    crop, l, q = _crop(psf_values, center)
    crop = np.array(crop, dtype=np.float64, order="C")  # writable copy for torch
    rows, cols = crop.shape[-2:]
    P = torch.from_numpy(crop).to(X.device)
    Y = torch.empty_like(X)
    batch, m, n = X.shape
    bcode = KB_BC_REFLECTIVE if bc_name(bc) == "reflective" else KB_BC_ZERO
    rc = load_library().kb_blur_direct(
        _ptr(P), rows * cols if per_image else 0, rows, cols, l, q, _ptr(X), _ptr(Y),
        m, n, batch, bcode, _stream_handle())
    _check(rc, "kb_blur_direct")
    return Y


def blur_direct(psf, X, bc):
    """Blur X by the PSF (psf.py:170-193): same arguments, errors and result as the reference.

    ``X`` may be a numpy array (returns a new float64 numpy array) or a CUDA torch tensor (returns
    a float64 CUDA tensor; no host copies)."""
    torch = _torch()
    on_device = isinstance(X, torch.Tensor)
    if on_device:
        if X.ndim != 2:
            raise ArgumentError("image must be 2-D")
        Xd = X.to(dtype=torch.float64).contiguous()
    else:
        Xh = np.asarray(X, dtype=float)
        if Xh.ndim != 2:
            raise ArgumentError("image must be 2-D")
        Xd = torch.from_numpy(np.ascontiguousarray(Xh)).to("cuda")
    m, n = Xd.shape
    rows, cols = psf.shape
    if rows > m or cols > n:
        raise ArgumentError(f"PSF of shape {psf.shape} larger than image {(m, n)}")
    Y = _launch(np.asarray(psf.values, dtype=np.float64), psf.center, Xd[None], bc, False)[0]
    if on_device:
        return Y
    return Y.cpu().numpy()


def blur_direct_batch(psfs, X, bc):
    """Blur each image X[k] ((batch, m, n) CUDA tensor) by its own PSF psfs[k] in one launch.

    The PSFs must share shape and centre (cfg3's per-image kernels); the result equals
    ``blur_direct(psfs[k], X[k], bc)`` image by image, bit for bit."""
    torch = _torch()
    if not isinstance(X, torch.Tensor) or X.ndim != 3:
        raise ArgumentError("expected a (batch, m, n) tensor")
    if len(psfs) != X.shape[0]:
        raise ArgumentError(f"{len(psfs)} PSFs for {X.shape[0]} images")
    shapes = {tuple(p.shape) for p in psfs}
    centers = {tuple(p.center) for p in psfs}
    if len(shapes) != 1 or len(centers) != 1:
        raise ArgumentError("batched PSFs must share shape and centre")
    rows, cols = shapes.pop()
    m, n = X.shape[1:]
    if rows > m or cols > n:
        raise ArgumentError(f"PSF of shape {(rows, cols)} larger than image {(m, n)}")
    vals = np.stack([np.asarray(p.values, dtype=np.float64) for p in psfs])
    return _launch(vals, centers.pop(), X.to(dtype=torch.float64).contiguous(), bc, True)
