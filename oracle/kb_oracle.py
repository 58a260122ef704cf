"""ctypes binding of oracle/libkb_oracle.so (kb_oracle.c) -- TEST INFRASTRUCTURE ONLY.

The direct banded fp64 restatement of the reference hot path (see kb_oracle.c for the file:line
map). Used by tests/ as the checker at BASELINE sizes where the numpy FFT port is too slow, and
by tests/golden/make_fullsize.py to generate full-length fixtures offline. Pinned by
tests/test_oracle_c.py against the numpy port (itself pinned to the reference's own outputs),
against the reference's cfg1 solution (tests/golden/cfg1.npz) and bit for bit against the
dense index rules on integer data.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "libkb_oracle.so")
_lib = None

_dp = ctypes.POINTER(ctypes.c_double)


class _Op(ctypes.Structure):
    _fields_ = [("m", ctypes.c_int), ("n", ctypes.c_int), ("r", ctypes.c_int), ("bc_a", ctypes.c_int),
                ("bc_b", ctypes.c_int), ("a_dlo", ctypes.c_int), ("a_w", ctypes.c_int), ("a_taps", _dp),
                ("b_dlo", ctypes.c_int), ("b_w", ctypes.c_int), ("b_taps", _dp)]


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            subprocess.run(["make", "-s", "-C", HERE], check=True)
        L = ctypes.CDLL(LIB)
        L.kbo_apply.argtypes = [ctypes.POINTER(_Op), ctypes.c_int, _dp, _dp]
        L.kbo_sfista.argtypes = [ctypes.POINTER(_Op), _dp, _dp, ctypes.c_double, ctypes.c_double, ctypes.c_int,
                                 _dp, ctypes.c_int, _dp]
        L.kbo_sfista.restype = ctypes.c_int
        L.kbo_power.argtypes = [ctypes.POINTER(_Op), _dp, ctypes.c_int, _dp, _dp, _dp]
        L.kbo_blur_direct.argtypes = [_dp, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, _dp,
                                      ctypes.c_int, ctypes.c_int, ctypes.c_int, _dp]
        L.kbo_threads.restype = ctypes.c_int
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(_dp)


def _kind(f) -> str:
    return getattr(f.kind, "value", f.kind)


def factor_band(f, rel_tol: float = 1e-14):
    """(dlo, taps) of a factor in stencil form: taps[t] = c_{dlo+t} = c[j + dlo + t] (1-based
    generator index, structured.py:111-123), cut to the entries above rel_tol * max|c| (exact
    zeros always; SURVEY F6 leakage on reflective generators)."""
    c = np.asarray(f.c, dtype=float)
    j = int(f.j)
    mag = np.abs(c)
    peak = mag.max() if c.size else 0.0
    keep = np.nonzero(mag > rel_tol * peak)[0] if peak > 0 else np.array([j - 1])
    lo, hi = int(keep.min()), int(keep.max())
    return lo - (j - 1), c[lo:hi + 1].copy()


class OracleOp:
    """Band tables of a KronOperator (reference-built or B200-built: reads t.H/t.K .c/.j/.kind).
    dtype "float32" rounds the taps to fp32 first (fp32-mode runs compare against an fp64 oracle
    fed the same fp32-rounded inputs)."""

    def __init__(self, op, dtype: str = "float64", rel_tol: float = 1e-14):
        self.shape = tuple(int(s) for s in op.shape)
        m, n = self.shape
        r = len(op.terms)

        def axis(factors):
            kinds = {_kind(f) for f in factors}
            if len(kinds) != 1 or kinds - {"toeplitz", "toeplitz_plus_hankel"}:
                raise ValueError(f"unsupported factor kinds {kinds}")
            bands = [factor_band(f, rel_tol) for f in factors]
            dlo = min(b[0] for b in bands)
            dhi = max(b[0] + b[1].size - 1 for b in bands)
            taps = np.zeros((len(bands), dhi - dlo + 1))
            for i, (lo, t) in enumerate(bands):
                taps[i, lo - dlo: lo - dlo + t.size] = t
            if dtype == "float32":
                taps = taps.astype(np.float32).astype(np.float64)
            return dlo, np.ascontiguousarray(taps), int(kinds == {"toeplitz_plus_hankel"})

        self.a_dlo, self.a_taps, self.bc_a = axis([t.H for t in op.terms])
        self.b_dlo, self.b_taps, self.bc_b = axis([t.K for t in op.terms])
        self.c = _Op(m, n, r, self.bc_a, self.bc_b, self.a_dlo, self.a_taps.shape[1], _p(self.a_taps),
                     self.b_dlo, self.b_taps.shape[1], _p(self.b_taps))


def apply(oop: OracleOp, X, adjoint: bool = False) -> np.ndarray:
    X = np.ascontiguousarray(X, dtype=np.float64)
    assert X.shape == oop.shape
    Y = np.empty_like(X)
    lib().kbo_apply(ctypes.byref(oop.c), int(adjoint), _p(X), _p(Y))
    return Y


def sfista(oop: OracleOp, B, L: float, lam: float, iters: int, beta, X0=None, project: bool = True,
           k0: int = 0) -> np.ndarray:
    """x_{k0+iters} of the projected engine from x_{k0} = X0 (y_{k0+1} = X0 only when k0 = 0)."""
    B = np.ascontiguousarray(B, dtype=np.float64)
    X = np.zeros_like(B) if X0 is None else np.array(X0, dtype=np.float64, order="C")
    work = np.empty((3,) + B.shape)
    beta = np.ascontiguousarray(np.asarray(beta, dtype=np.float64)[k0:k0 + iters])
    bad = lib().kbo_sfista(ctypes.byref(oop.c), _p(B), _p(X), float(L), float(lam), int(iters), _p(beta),
                           int(bool(project)), _p(work))
    if bad:
        raise FloatingPointError(f"non-finite iterate at iteration {k0 + bad}")
    return X


def power(oop: OracleOp, v0, iters: int):
    """(rho[iters], ||w||^2[iters]) of the matrix-form power iteration from the normalised v0."""
    v = np.array(v0, dtype=np.float64, order="C")
    rho, nw2 = np.zeros(iters), np.zeros(iters)
    work = np.empty((2,) + v.shape)
    lib().kbo_power(ctypes.byref(oop.c), _p(v), int(iters), _p(rho), _p(nw2), _p(work))
    return rho, nw2


def blur_direct(values, center, X, bc: str) -> np.ndarray:
    P = np.ascontiguousarray(values, dtype=np.float64)
    X = np.ascontiguousarray(X, dtype=np.float64)
    Y = np.empty_like(X)
    lib().kbo_blur_direct(_p(P), P.shape[0], P.shape[1], int(center[0]), int(center[1]), _p(X), X.shape[0],
                          X.shape[1], 1 if bc == "reflective" else 0, _p(Y))
    return Y


def threads() -> int:
    return int(lib().kbo_threads())
