"""numpy port of the kronblur hot path (test oracle / CPU baseline; see oracle/__init__.py).

Every function cites the reference lines it restates. Factors are any objects with ``c`` (length-n
generator), ``j`` (1-based anchor), ``n`` and ``kind`` (enum or str: toeplitz / hankel /
toeplitz_plus_hankel); operators are any objects with ``terms`` (each with ``H``, ``K``) and
``shape`` — so the port runs on reference-built and B200-package-built operators alike.
"""

from __future__ import annotations

import warnings
from concurrent.futures import ThreadPoolExecutor

import numpy as np

DENSE_FFT_CROSSOVER = 128  # structured.py:41
LIPSCHITZ_SAFETY = 1.05    # solvers.py:43


def _kind(f) -> str:
    return getattr(f.kind, "value", f.kind)


# ---------------------------------------------------------------- dense index rules
def dense_toeplitz(c, j: int) -> np.ndarray:
    """T[i,k] = c[j+i-k] for 1 <= j+i-k <= n (structured.py:111-115)."""
    c = np.asarray(c, dtype=float)
    n = c.size
    T = np.zeros((n, n))
    for d in range(1 - j, n - j + 1):  # diagonal offset i-k carries c[j+d]
        val = c[j + d - 1]
        if d >= 0:
            idx = np.arange(d, n)
            T[idx, idx - d] = val
        else:
            idx = np.arange(0, n + d)
            T[idx, idx - d] = val
    return T


def dense_hankel(c, j: int) -> np.ndarray:
    """H[i,k] = c[i+k+j-1] (<= n) or c[i+k+j-1-2n] (1..j-1) (structured.py:118-123)."""
    c = np.asarray(c, dtype=float)
    n = c.size
    i = np.arange(1, n + 1)[:, None]
    k = np.arange(1, n + 1)[None, :]
    s = i + k + j - 1
    H = np.zeros((n, n))
    top = s <= n
    H[top] = c[(s[top] - 1)]
    w = s - 2 * n
    bot = (w >= 1) & (w <= j - 1)
    H[bot] = c[w[bot] - 1]
    return H


def dense_factor(f) -> np.ndarray:
    kind = _kind(f)
    if kind == "toeplitz":
        return dense_toeplitz(f.c, f.j)
    if kind == "hankel":
        return dense_hankel(f.c, f.j)
    return dense_toeplitz(f.c, f.j) + dense_hankel(f.c, f.j)


# ---------------------------------------------------------------- FFT apply (structured.py)
def _fft_len(n: int) -> int:
    """Power of two >= 2n-1 (structured.py:99)."""
    return 1 << (2 * n - 2).bit_length() if n > 1 else 1


def _toeplitz_symbol(c, j: int, length: int) -> np.ndarray:
    """Circulant first column carrying diagonal d = i-k at position d mod length (structured.py:74-80)."""
    n = c.size
    col = np.zeros(length)
    col[np.mod(np.arange(n) - (j - 1), length)] = c
    return col


def _hankel_reversed_symbol(c, j: int, length: int) -> np.ndarray:
    """Circulant column of H with reversed columns (structured.py:83-94)."""
    n = c.size
    col = np.zeros(length)
    d = np.arange(1 - n, 1 - j)  # d in [1-n, -j]
    col[np.mod(d, length)] = c[d + n + j - 1]
    if j >= 2:
        d2 = np.arange(n + 1 - j, n)
        col[np.mod(d2, length)] = c[d2 + j - n - 1]
    return col


class FactorPlan:
    """Spectra of one factor for the FFT apply (structured.py:97-108), cached per factor."""

    def __init__(self, f):
        c = np.asarray(f.c, dtype=float)
        self.n = c.size
        self.length = _fft_len(self.n)
        kind = _kind(f)
        self.t_hat = np.fft.rfft(_toeplitz_symbol(c, f.j, self.length)) if kind != "hankel" else None
        self.h_hat = np.fft.rfft(_hankel_reversed_symbol(c, f.j, self.length)) if kind != "toeplitz" else None
        self.dense = dense_factor(f) if self.n < DENSE_FFT_CROSSOVER else None


_pool = None
_threads = 1


def set_threads(n: int) -> None:
    """Column-block threading of the FFT apply (numpy's FFT releases the GIL). Columns are
    transformed independently, so results are bit-identical for any thread count."""
    global _pool, _threads
    n = max(1, int(n))
    if n != _threads:
        if _pool is not None:
            _pool.shutdown()
        _pool = ThreadPoolExecutor(max_workers=n) if n > 1 else None
        _threads = n


def factor_apply(plan: FactorPlan, X: np.ndarray, transpose: bool = False) -> np.ndarray:
    """F X or F^T X for an n x p block (structured.py:179-228)."""
    if _pool is not None and plan.dense is None and X.shape[1] >= 2 * _threads:
        edges = np.linspace(0, X.shape[1], _threads + 1).astype(int)
        parts = list(_pool.map(lambda ab: _factor_apply(plan, X[:, ab[0]:ab[1]], transpose),
                               zip(edges[:-1], edges[1:])))
        return np.concatenate(parts, axis=1)
    return _factor_apply(plan, X, transpose)


def _factor_apply(plan: FactorPlan, X: np.ndarray, transpose: bool) -> np.ndarray:
    if plan.dense is not None:
        return plan.dense.T @ X if transpose else plan.dense @ X
    n, L = plan.n, plan.length
    out = np.zeros_like(X)
    buf = np.zeros((L, X.shape[1]))
    if plan.t_hat is not None:
        sym = np.conj(plan.t_hat) if transpose else plan.t_hat
        buf[:n] = X
        out += np.fft.irfft(np.fft.rfft(buf, axis=0) * sym[:, None], n=L, axis=0)[:n]
    if plan.h_hat is not None:  # Hankel is symmetric: transpose reuses the spectrum
        buf[:n] = X[::-1]
        out += np.fft.irfft(np.fft.rfft(buf, axis=0) * plan.h_hat[:, None], n=L, axis=0)[:n]
    return out


class PortOperator:
    """Plans for every factor of a KronOperator."""

    def __init__(self, op):
        self.shape = tuple(op.shape)
        self.plans = [(FactorPlan(t.H), FactorPlan(t.K)) for t in op.terms]


def kron_apply(pop: PortOperator, X: np.ndarray) -> np.ndarray:
    """sum_i H_i X K_i^T, sequential in-order sum (kron.py:218-225)."""
    X = np.asarray(X, dtype=float)
    Y = np.zeros_like(X)
    for ph, pk in pop.plans:
        Z = factor_apply(ph, X)
        Y += factor_apply(pk, Z.T).T
    return Y


def kron_apply_adjoint(pop: PortOperator, Y: np.ndarray) -> np.ndarray:
    """sum_i H_i^T Y K_i (kron.py:228-235)."""
    Y = np.asarray(Y, dtype=float)
    X = np.zeros_like(Y)
    for ph, pk in pop.plans:
        Z = factor_apply(ph, Y, transpose=True)
        X += factor_apply(pk, Z.T, transpose=True).T
    return X


def dense_kron_apply(op, X, adjoint: bool = False) -> np.ndarray:
    """Same operator through materialised factors (exact on integer data)."""
    X = np.asarray(X, dtype=float)
    Y = np.zeros_like(X)
    for t in op.terms:
        Hd, Kd = dense_factor(t.H), dense_factor(t.K)
        if adjoint:
            Y += Hd.T @ X @ Kd
        else:
            Y += Hd @ X @ Kd.T
    return Y


# ---------------------------------------------------------------- solver pieces
def momentum_next(t: float) -> float:
    """(1 + sqrt(1 + 4 t^2)) / 2 (solvers.py:96-101)."""
    t = float(t)
    if not (np.isfinite(t) and t >= 1.0):
        raise ValueError(f"momentum parameter must be >= 1, got {t}")
    return (1.0 + np.sqrt(1.0 + 4.0 * t * t)) / 2.0


def lipschitz_start(seed: int, shape) -> np.ndarray:
    """Normalised Philox start vector of solvers.py:115-120 (rand.py:26-36)."""
    key = (4, 0)  # rand.py:22 "lipschitz" tag, primary stream
    rng = np.random.Generator(np.random.Philox(np.random.SeedSequence(entropy=int(seed), spawn_key=key)))
    v = rng.standard_normal(shape)
    return v / np.linalg.norm(v.ravel())


def estimate_lipschitz(apply, apply_adjoint, dims, iters: int = 50, seed: int = 0) -> float:
    """Power iteration on A^T A times 1.05 (solvers.py:104-130)."""
    shape = (dims,) if np.isscalar(dims) else tuple(dims)
    v = lipschitz_start(seed, shape)
    rho = 0.0
    for _ in range(int(iters)):
        w = apply_adjoint(apply(v))
        rho = float(np.vdot(v.ravel(), w.ravel()))
        nw = np.linalg.norm(w.ravel())
        if nw == 0 or rho <= 0:
            warnings.warn("operator is numerically zero; Lipschitz floor returned")
            return float(np.finfo(float).eps)
        v = w / nw
    return LIPSCHITZ_SAFETY * rho


def engine(apply, apply_adjoint, b, L: float, lam: float, iters: int, x0=None,
           project: bool = False, record_iterates: bool = False):
    """The _engine loop (solvers.py:153-199) without history; optional x >= 0 after :171.

    Returns (x_last, iterates). Raises FloatingPointError("non-finite iterate at iteration k").
    """
    b = np.asarray(b, dtype=float)
    x_prev = np.zeros_like(b) if x0 is None else np.array(x0, dtype=float)
    denom = L + lam**2
    y = x_prev
    t = 1.0
    iterates = []
    for k in range(1, int(iters) + 1):
        grad = apply_adjoint(apply(y) - b)
        x = (L * y - grad) / denom
        if project:
            x = np.maximum(x, 0.0)
        t_next = momentum_next(t)
        y = x + ((t - 1.0) / t_next) * (x - x_prev)
        if not np.all(np.isfinite(x)):
            raise FloatingPointError(f"non-finite iterate at iteration {k}")
        if record_iterates:
            iterates.append(x.copy())
        x_prev = x
        t = t_next
    return x_prev, iterates


def sfista(op, B, L: float, lam: float, iters: int, X0=None, project: bool = False,
           record_iterates: bool = False):
    """Matrix-form solve on the port operator (solvers.py:215-228 + projection)."""
    pop = op if isinstance(op, PortOperator) else PortOperator(op)
    return engine(lambda Y: kron_apply(pop, Y), lambda Y: kron_apply_adjoint(pop, Y), B, L, lam,
                  iters, X0, project, record_iterates)


# ---------------------------------------------------------------- exact blur
def blur_direct(values, center, X, bc: str) -> np.ndarray:
    """Shifted-copy blur, psf.py:170-193: pad by ((rows-l, l-1), (cols-q, q-1)) with zeros or
    numpy "symmetric" mode (:184-186), then Y += P[a0, b0] * Xp[rows-1-a0 : +m, cols-1-b0 : +n] over
    np.nonzero(P) in row-major order (:187-192)."""
    P = np.asarray(values, dtype=float)
    X = np.asarray(X, dtype=float)
    m, n = X.shape
    rows, cols = P.shape
    l, q = int(center[0]), int(center[1])
    pad = ((rows - l, l - 1), (cols - q, q - 1))
    Xp = np.pad(X, pad, mode="constant" if bc == "zero" else "symmetric")
    Y = np.zeros_like(X)
    for a0, b0 in zip(*np.nonzero(P)):
        r0, c0 = rows - 1 - a0, cols - 1 - b0
        Y += P[a0, b0] * Xp[r0 : r0 + m, c0 : c0 + n]
    return Y


def blur_direct_pixel(values, center, X, bc: str, i: int, j: int) -> float:
    """One output pixel of blur_direct by the same per-pixel sequence (separately rounded products
    and sums over the nonzeros in row-major order): for sampled checks at sizes where the whole
    image would take hours in numpy."""
    P = np.asarray(values, dtype=float)
    m, n = X.shape
    l, q = int(center[0]), int(center[1])

    def ext(t, M):
        if 0 <= t < M:
            return t
        if bc == "zero":
            return -1
        return -1 - t if t < 0 else 2 * M - 1 - t

    y = 0.0
    for a0, b0 in zip(*np.nonzero(P)):
        gi, gj = ext(i + l - 1 - a0, m), ext(j + q - 1 - b0, n)
        x = float(X[gi, gj]) if gi >= 0 and gj >= 0 else 0.0
        y = y + float(P[a0, b0]) * x
    return y


# ---------------------------------------------------------------- lambda selection
def select_lambda(op, B, noise_level: float, lipschitz: float, grid_points: int = 25,
                  probe_iters: int = 50, dense_limit: int = 1024, probe_terms: int = 5):
    """Discrepancy-principle lambda, solvers.py:255-306: log grid [1e-4, 1] * sqrt(L) (:281-282),
    target noise_level * ||vec B|| (:283-284), dense eigen route for m n <= 1024 (:286-293),
    else 50-iteration sFISTA probes on the first min(5, r) terms (:294-305). Returns
    (lambda, residuals)."""
    B = np.asarray(B, dtype=float)
    scale = np.sqrt(lipschitz)
    grid = np.geomspace(1e-4 * scale, scale, int(grid_points))
    b = B.flatten(order="F")
    target = noise_level * np.linalg.norm(b)
    m, n = B.shape
    residuals = np.empty(grid.size)
    if m * n <= dense_limit:
        A = sum(np.kron(dense_factor(t.K), dense_factor(t.H)) for t in op.terms)
        w, Q = np.linalg.eigh(A.T @ A)
        z = Q.T @ (A.T @ b)
        bb = float(b @ b)
        for i, lam in enumerate(grid):
            xh = z / (w + lam**2)
            residuals[i] = np.sqrt(max(bb - 2.0 * float(z @ xh) + float((w * xh) @ xh), 0.0))
    else:
        pop = PortOperator(type("Probe", (), {"terms": list(op.terms)[:min(probe_terms, len(op.terms))],
                                              "shape": tuple(op.shape)})())
        for i, lam in enumerate(grid):
            x, _ = sfista(pop, B, lipschitz, float(lam), int(probe_iters))
            residuals[i] = np.linalg.norm(kron_apply(pop, x) - B)
    return float(grid[int(np.argmin(np.abs(residuals - target)))]), residuals
