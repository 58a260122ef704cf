"""Banded Toeplitz / Toeplitz+Hankel factors (restates the data model of kronblur structured.py).

The reference stores every factor as a full-length generator ``c`` (length n) with a 1-based band
anchor ``j`` and applies it through a circulant FFT embedding (structured.py:97-108, 184-198). The
B200 path never builds spectra: it extracts the band of nonzero stencil taps

    c_d = c[j + d]      (1-based c, offsets d = 1-j .. n-j)

so that F x is the stencil y[s] = sum_d c_d * x~(s - d) with x~ the zero (TOEPLITZ) or single
half-sample reflected (TOEPLITZ_PLUS_HANKEL) extension of x — identical to the index rules
T[i,k] = c[j+i-k] and H[i,k] = c[i+k+j-1] / c[i+k+j-1-2n] of structured.py:111-123. The band is
uploaded once per operator (``device.DeviceOperator``).
"""

from __future__ import annotations

import enum
from dataclasses import dataclass, field

import numpy as np

from .errors import ArgumentError, CapacityError

DENSE_GUARD = 4096  # structured.py:44


class FactorKind(enum.Enum):
    TOEPLITZ = "toeplitz"
    HANKEL = "hankel"
    TOEPLITZ_PLUS_HANKEL = "toeplitz_plus_hankel"


@dataclass(frozen=True)
class StructuredFactor:
    """Immutable banded factor (structured.py:62-71 minus the FFT plan)."""

    kind: FactorKind
    c: np.ndarray = field(repr=False)
    j: int
    n: int


def _make(kind: FactorKind, c, j: int) -> StructuredFactor:
    c = np.array(c, dtype=float)
    if c.ndim != 1 or c.size == 0:
        raise ArgumentError("generator must be a nonempty 1-D vector")
    if not np.all(np.isfinite(c)):
        raise ArgumentError("generator has non-finite entries")
    j = int(j)
    if not 1 <= j <= c.size:
        raise ArgumentError(f"band anchor j={j} outside 1..{c.size}")
    c.flags.writeable = False
    return StructuredFactor(kind=kind, c=c, j=j, n=c.size)


def toep(c, j: int) -> StructuredFactor:
    return _make(FactorKind.TOEPLITZ, c, j)


def hank(c, j: int) -> StructuredFactor:
    return _make(FactorKind.HANKEL, c, j)


def toep_plus_hank(c, j: int) -> StructuredFactor:
    return _make(FactorKind.TOEPLITZ_PLUS_HANKEL, c, j)


def kind_name(factor) -> str:
    return getattr(factor.kind, "value", factor.kind)


def factor_band(factor, rel_tol: float = 0.0) -> tuple[int, np.ndarray]:
    """Stencil band ``(dlo, taps)`` of a factor: taps[t] = c_{dlo+t} = c[j+dlo+t].

    Entries with |c| <= rel_tol * max|c| at either end are trimmed (``rel_tol=0`` keeps every
    nonzero, i.e. the band is exact). A zero generator yields the single tap c_0 = 0.
    """
    c = np.asarray(factor.c, dtype=float)
    j = int(factor.j)
    mag = np.abs(c)
    peak = float(mag.max()) if mag.size else 0.0
    keep = np.nonzero(mag > rel_tol * peak)[0] if peak > 0 else np.array([], dtype=int)
    if keep.size == 0:
        return 0, np.zeros(1)
    lo, hi = int(keep[0]), int(keep[-1])  # 0-based positions in c
    return lo + 1 - j, c[lo : hi + 1].copy()


def _dense_toeplitz(c: np.ndarray, j: int) -> np.ndarray:
    n = c.size
    i = np.arange(n)[:, None]
    k = np.arange(n)[None, :]
    idx = j + i - k  # 1-based generator index
    ok = (idx >= 1) & (idx <= n)
    return np.where(ok, c[np.clip(idx - 1, 0, n - 1)], 0.0)


def _dense_hankel(c: np.ndarray, j: int) -> np.ndarray:
    n = c.size
    s = np.arange(1, n + 1)[:, None] + np.arange(1, n + 1)[None, :] + j - 1
    direct = np.where(s <= n, c[np.clip(s - 1, 0, n - 1)], 0.0)
    w = s - 2 * n
    wrapped = (w >= 1) & (w <= j - 1)
    return np.where(wrapped, c[np.clip(w - 1, 0, n - 1)], direct)


def factor_to_dense(factor) -> np.ndarray:
    """Materialise a factor as n x n (guarded like structured.py:170-176); test/setup helper."""
    n = int(factor.n)
    if n > DENSE_GUARD:
        raise CapacityError(f"dense factor of order {n} exceeds guard {DENSE_GUARD}")
    c = np.asarray(factor.c, dtype=float)
    kind = kind_name(factor)
    if kind == "toeplitz":
        return _dense_toeplitz(c, factor.j)
    if kind == "hankel":
        return _dense_hankel(c, factor.j)
    return _dense_toeplitz(c, factor.j) + _dense_hankel(c, factor.j)
