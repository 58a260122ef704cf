"""PSF container, boundary conditions and padding (restates kronblur psf.py:35-167).

Only what the hot path's setup consumes: ``Psf`` validation, ``BoundaryCondition``, ``pad_to``
(which fixes the band anchor, psf.py:135-154) and the column-stacking ``vec``/``unvec`` pair used
by the vector-form callers (pipeline.py:117-122).
"""

from __future__ import annotations

import enum
from dataclasses import dataclass

import numpy as np

from .errors import ArgumentError


class BoundaryCondition(enum.Enum):
    ZERO = "zero"
    REFLECTIVE = "reflective"


def bc_name(bc) -> str:
    """'zero' / 'reflective' for this module's enum, the reference's enum, or a plain string."""
    value = getattr(bc, "value", bc)
    if value not in ("zero", "reflective"):
        raise ArgumentError(f"unknown boundary condition {bc!r}")
    return value


@dataclass(frozen=True)
class Psf:
    """Nonnegative kernel summing to one with a 1-based centre (l, q) (psf.py:40-68)."""

    values: np.ndarray
    center: tuple[int, int]

    def __post_init__(self):
        v = np.array(self.values, dtype=float)
        if v.ndim != 2 or v.size == 0:
            raise ArgumentError("PSF must be a nonempty 2-D array")
        if not np.all(np.isfinite(v)):
            raise ArgumentError("PSF has non-finite entries")
        if np.any(v < 0):
            raise ArgumentError("PSF entries must be nonnegative")
        total = float(v.sum())
        if abs(total - 1.0) > 1e-8:
            raise ArgumentError(f"PSF must sum to 1, got {total!r}")
        l, q = int(self.center[0]), int(self.center[1])
        if not (1 <= l <= v.shape[0] and 1 <= q <= v.shape[1]):
            raise ArgumentError(f"PSF center {(l, q)} outside array of shape {v.shape}")
        v.flags.writeable = False
        object.__setattr__(self, "values", v)
        object.__setattr__(self, "center", (l, q))

    @property
    def shape(self) -> tuple[int, int]:
        return self.values.shape


def pad_to(psf, m: int, n: int) -> Psf:
    """Zero-pad to m x n with the centre moved as close to the middle as the kernel allows.

    Same placement rule as psf.py:147-149: centre row = clamp(m//2+1, l, m-rows+l).
    """
    m, n = int(m), int(n)
    rows, cols = psf.values.shape
    if rows > m or cols > n:
        raise ArgumentError(f"cannot pad PSF of shape {psf.values.shape} to smaller {(m, n)}")
    l, q = psf.center
    lc = min(max(m // 2 + 1, l), m - rows + l)
    qc = min(max(n // 2 + 1, q), n - cols + q)
    out = np.zeros((m, n))
    out[lc - l : lc - l + rows, qc - q : qc - q + cols] = psf.values
    return Psf(out, (lc, qc))


def vec(X) -> np.ndarray:
    """Column stacking (Fortran order), psf.py:157-159."""
    return np.asarray(X, dtype=float).flatten(order="F")


def unvec(v, m: int, n: int) -> np.ndarray:
    """Inverse of ``vec`` (psf.py:162-167)."""
    v = np.asarray(v, dtype=float)
    if v.ndim != 1 or v.size != m * n:
        raise ArgumentError(f"expected a vector of length {m * n}, got shape {v.shape}")
    return v.reshape((m, n), order="F")
