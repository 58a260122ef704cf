"""Kronecker-sum operator: KPA setup on the host, application on the B200.

* ``decompose`` (reference kron.py:156-208) — the one-time setup, excluded from timing. Instead of
  the reference's full image-size SVD of the weighted PSF (O(n^3), ~15 min at 16384^2) it runs the
  *support-block* KPA: because the padded PSF is zero outside its support block S,
  the weighted SVD reduces to the SVD of the |S_r| x |S_c| core G_r P_S G_c^T, where G is the
  diagonal zero-BC weight (kron.py:89-103) or the upper Cholesky factor of the fold Gram matrix
  restricted to S (kron.py:106-126). The singular values are the same and the generators
  a_i = sqrt(sigma_i) G_r^{-1} u_i, embedded at S, satisfy the same orthogonality in the weighted
  inner product, so they agree with the reference's up to sign; signs are fixed by the rule
  "first entry above 1e-3 max|a| is positive". When more terms are requested than
  the block has, the full weighted SVD of the reference is used instead.
* ``kron_apply`` / ``kron_apply_adjoint`` (kron.py:218-235) run on the GPU through the C ABI.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import scipy.linalg

from .errors import ArgumentError, CapacityError, NumericError
from .psf import BoundaryCondition, Psf, bc_name, pad_to
from .structured import StructuredFactor, factor_to_dense, toep, toep_plus_hank

DENSE_OPERATOR_GUARD = 4096  # psf.py:30


@dataclass(frozen=True)
class KronTerm:
    sigma: float
    H: StructuredFactor
    K: StructuredFactor


def truncation_error(sigma, s: int) -> float:
    """||A - A_s||_F = sqrt(sum_{i>s} sigma_i^2) (kron.py:147-153)."""
    sigma = np.asarray(sigma, dtype=float)
    s = int(s)
    if not 0 <= s <= sigma.size:
        raise ArgumentError(f"s={s} outside 0..{sigma.size}")
    return float(np.sqrt(np.sum(sigma[s:] ** 2)))


@dataclass(frozen=True)
class KronOperator:
    """A_s = sum_i K_i (x) H_i for an m x n image (kron.py:61-86)."""

    terms: tuple
    shape: tuple
    bc: BoundaryCondition
    sigma: np.ndarray = field(repr=False)
    s: int
    rank: int
    eps: float

    def truncate(self, s: int) -> "KronOperator":
        s = int(s)
        if not 1 <= s <= len(self.terms):
            raise ArgumentError(f"s={s} outside 1..{len(self.terms)}")
        return KronOperator(
            terms=self.terms[:s], shape=self.shape, bc=self.bc, sigma=self.sigma, s=s,
            rank=self.rank, eps=truncation_error(self.sigma, s),
        )


def _axis_weights(n: int, center: int) -> np.ndarray:
    """Zero-BC weights sqrt(n - |i - l|), i = 1..n (kron.py:89-91)."""
    return np.sqrt(n - np.abs(np.arange(1, n + 1) - center))


def _fold_gram(n: int) -> np.ndarray:
    """Gram of Toeplitz+Hankel columns: n on the diagonal, 1 at odd lags (kron.py:106-112)."""
    first = np.zeros(n)
    first[0] = float(n)
    first[1::2] = 1.0
    return scipy.linalg.toeplitz(first)


def _support(v: np.ndarray, axis: int) -> np.ndarray:
    nz = np.nonzero(np.any(v != 0, axis=axis))[0]
    if nz.size == 0:
        return np.arange(1)
    return np.arange(nz[0], nz[-1] + 1)


def _sign_fix(a: np.ndarray, b: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    mag = np.abs(a)
    peak = mag.max()
    if peak > 0:
        first = int(np.argmax(mag > 1e-3 * peak))
        if a[first] < 0:
            return -a, -b
    return a, b


def _weighting(bc: str, m: int, n: int, l: int, q: int, rows: np.ndarray, cols: np.ndarray):
    """Row/column maps (G, solve) restricted to index sets rows/cols."""
    if bc == "zero":
        wr = _axis_weights(m, l)[rows]
        wc = _axis_weights(n, q)[cols]
        return (lambda P: wr[:, None] * P * wc[None, :],
                lambda u: u / wr, lambda v: v / wc)
    try:
        gr = np.linalg.cholesky(_fold_gram(m)[np.ix_(rows, rows)]).T
        gc = gr if (n == m and np.array_equal(rows, cols)) else np.linalg.cholesky(
            _fold_gram(n)[np.ix_(cols, cols)]).T
    except np.linalg.LinAlgError as exc:  # pragma: no cover - Gram blocks are SPD
        raise NumericError(f"fold Gram factorization failed: {exc}") from exc
    return (lambda P: gr @ P @ gc.T,
            lambda u: scipy.linalg.solve_triangular(gr, u, lower=False),
            lambda v: scipy.linalg.solve_triangular(gc, v, lower=False))


def decompose(psf, bc, s: int | None = None, shape: tuple | None = None) -> KronOperator:
    """s-term weighted-SVD Kronecker expansion of the blur operator (kron.py:156-208)."""
    if shape is not None:
        psf = pad_to(psf, shape[0], shape[1])
    P = np.asarray(psf.values, dtype=float)
    m, n = P.shape
    l, q = psf.center
    name = bc_name(bc)
    if m != n:
        raise ArgumentError(f"weighting needs a square PSF, got {m}x{n}; pad first")
    if s is not None and not 1 <= int(s) <= min(m, n):
        raise ArgumentError(f"s={s} outside 1..{min(m, n)}")

    rows = _support(P, axis=1)
    cols = _support(P, axis=0)
    block = s is None or int(s) <= min(rows.size, cols.size)
    if not block:  # full weighted SVD, as the reference does
        rows = np.arange(m)
        cols = np.arange(n)
    core_of, back_r, back_c = _weighting(name, m, n, l, q, rows, cols)
    core = core_of(P[np.ix_(rows, cols)])
    if not np.all(np.isfinite(core)):
        raise ArgumentError("SVD input has non-finite entries")
    try:
        U, sig, Vt = np.linalg.svd(core, full_matrices=False)
    except np.linalg.LinAlgError as exc:
        raise NumericError(f"SVD failed to converge: {exc}") from exc
    sigma = np.zeros(min(m, n))
    sigma[: sig.size] = sig
    cutoff = sigma[0] * max(m, n) * np.finfo(float).eps
    rank = int(np.count_nonzero(sigma > cutoff))
    if s is None:
        s = max(rank, 1)
        if s > min(rows.size, cols.size):  # pragma: no cover - rank <= block size
            raise ArgumentError("rank exceeds support block")
    s = int(s)

    make = toep if name == "zero" else toep_plus_hank
    terms = []
    for i in range(s):
        root = np.sqrt(sig[i])
        a = np.zeros(m)
        b = np.zeros(n)
        a[rows] = root * back_r(U[:, i])
        b[cols] = root * back_c(Vt[i, :])
        a, b = _sign_fix(a, b)
        terms.append(KronTerm(sigma=float(sig[i]), H=make(a, l), K=make(b, q)))
    sigma.flags.writeable = False
    enum_bc = bc if isinstance(bc, BoundaryCondition) else BoundaryCondition(name)
    return KronOperator(terms=tuple(terms), shape=(m, n), bc=enum_bc, sigma=sigma, s=s,
                        rank=rank, eps=truncation_error(sigma, s))


def kron_to_dense(op) -> np.ndarray:
    """Materialise A_s (guarded; test helper, kron.py:238-246)."""
    m, n = op.shape
    if m * n > DENSE_OPERATOR_GUARD:
        raise CapacityError(f"dense operator of size {m * n} exceeds guard {DENSE_OPERATOR_GUARD}")
    A = np.zeros((m * n, m * n))
    for t in op.terms:
        A += np.kron(factor_to_dense(t.K), factor_to_dense(t.H))
    return A


def _check_image(op, X):
    import torch

    if isinstance(X, torch.Tensor):
        if tuple(X.shape) != tuple(op.shape):
            raise ArgumentError(f"image shape {tuple(X.shape)} does not match operator shape {tuple(op.shape)}")
        return X
    X = np.asarray(X, dtype=float)
    if X.shape != tuple(op.shape):
        raise ArgumentError(f"image shape {X.shape} does not match operator shape {tuple(op.shape)}")
    return X


def _apply(op, X, adjoint: bool, dtype: str | None):
    import torch

    from .device import device_operator

    X = _check_image(op, X)
    if isinstance(X, torch.Tensor) and X.is_cuda:
        dt = dtype or ("float32" if X.dtype == torch.float32 else "float64")
        dev = device_operator(op, dt)
        return dev.apply(X.to(dev.tdtype).contiguous(), adjoint=adjoint)
    dev = device_operator(op, dtype or "float64")
    with dev.exclusive():
        d_in = dev.staging("apply_in")
        d_in.copy_(torch.from_numpy(np.ascontiguousarray(X)).to(dev.tdtype), non_blocking=False)
        out = dev.apply(d_in, out=dev.staging("apply_out"), adjoint=adjoint)
        return out.to("cpu", torch.float64).numpy().copy()


def kron_apply(op, X, *, dtype: str | None = None):
    """A_s X = sum_i H_i X K_i^T on the GPU (kron.py:218-225). numpy in -> numpy fp64 out;
    a CUDA tensor in -> CUDA tensor out."""
    return _apply(op, X, False, dtype)


def kron_apply_adjoint(op, Y, *, dtype: str | None = None):
    """A_s^T Y = sum_i H_i^T Y K_i on the GPU (kron.py:228-235)."""
    return _apply(op, Y, True, dtype)
