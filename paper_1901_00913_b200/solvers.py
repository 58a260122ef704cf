"""sFISTA on the B200 behind the reference solver API (kronblur solvers.py).

``sfista(op, B, cfg, X0=None, truth=None, exact_apply=None)`` keeps the reference signature and
``SolveRun`` result (solvers.py:215-228). Its loop is the reference ``_engine`` (solvers.py:153-199)
executed by the native runner ``kb_sfista_run``: per iteration one fused forward kernel pair
(R = A y - B) and one fused adjoint+update pair (x = (L y - A^T R)/(L + lam^2), optional x >= 0
projection, y = x + beta_k (x - x_prev)). The momentum coefficients beta_k are data independent and
come from ``momentum_next`` on the host, bit-identical to the reference recurrence.

Extensions (keyword-only, so the reference signature is unchanged): ``options=SolveOptions(...)``
selects the compute dtype (float64 / float32), the x >= 0 projection that BASELINE's configs ask
for (the reference has none), and CUDA-graph use.

Semantics kept from the reference:
  * X0 shape mismatch -> ArgumentError (:155-157); y_1 = X0, t_1 = 1 (:160-161)
  * non-finite x_k -> NumericError("non-finite iterate at iteration k") (:175-176)
  * record_history: IterationRecord(k, t_k, Phi_s(x_k), eta, gamma, cumulative ms) (:180-192);
    record_iterates: a copy of every x_k (:193-194); rel_tol early stop (:197-198)
  * solve_ms covers only the iteration bodies (:169-174), here timed with CUDA events.
"""

from __future__ import annotations

import functools
import warnings
from dataclasses import dataclass, field

import numpy as np

from .errors import ArgumentError, NumericError

LIPSCHITZ_SAFETY = 1.05  # solvers.py:43


@dataclass(frozen=True)
class SolveConfig:
    """Solver parameters (solvers.py:53-72)."""

    lam: float
    lipschitz: float
    max_iter: int = 50
    rel_tol: float = 0.0
    record_history: bool = True
    record_iterates: bool = False

    def __post_init__(self):
        if not (np.isfinite(self.lam) and self.lam > 0):
            raise ArgumentError(f"lambda must be positive, got {self.lam}")
        if not (np.isfinite(self.lipschitz) and self.lipschitz > 0):
            raise ArgumentError(f"Lipschitz constant must be positive, got {self.lipschitz}")
        if self.max_iter < 1:
            raise ArgumentError(f"max_iter must be >= 1, got {self.max_iter}")
        if self.rel_tol < 0:
            raise ArgumentError(f"rel_tol must be >= 0, got {self.rel_tol}")


@dataclass(frozen=True)
class IterationRecord:
    k: int
    t: float
    objective: float
    eta: float | None
    gamma: float | None
    ms: float


@dataclass
class SolveRun:
    x: np.ndarray
    iterations: int
    solve_ms: float
    history: list = field(default_factory=list)
    iterates: list = field(default_factory=list)


@dataclass(frozen=True)
class SolveOptions:
    """B200-specific knobs (not part of the reference signature)."""

    dtype: str = "float64"     # compute dtype of the device planes
    project: bool = False      # x >= 0 after the update (BASELINE configs); reference has none
    use_graph: bool | None = None  # None: graph when the fast path runs >= 8 iterations


def momentum_next(t: float) -> float:
    """t_{k+1} = (1 + sqrt(1 + 4 t^2)) / 2 (solvers.py:96-101)."""
    t = float(t)
    if not (np.isfinite(t) and t >= 1.0):
        raise ArgumentError(f"momentum parameter must be >= 1, got {t}")
    return (1.0 + np.sqrt(1.0 + 4.0 * t * t)) / 2.0


def momentum_table(iters: int) -> tuple[np.ndarray, np.ndarray]:
    """(t_k for k=1..iters, beta_k = (t_k - 1)/t_{k+1}) exactly as _engine evaluates them.
    Data-independent, so computed once per length (read-only arrays; ~2 us per scalar step)."""
    return _momentum_cached(int(iters))


@functools.lru_cache(maxsize=64)
def _momentum_cached(iters: int) -> tuple[np.ndarray, np.ndarray]:
    ts = np.empty(iters)
    beta = np.empty(iters)
    t = 1.0
    for k in range(iters):
        tn = momentum_next(t)
        ts[k] = t
        beta[k] = (t - 1.0) / tn
        t = tn
    ts.flags.writeable = False
    beta.flags.writeable = False
    return ts, beta


def objective(apply, x, b, lam: float) -> float:
    """Phi(x) = 1/2 ||A x - b||^2 + lam^2/2 ||x||^2 over raveled arrays (solvers.py:133-141)."""
    r = np.asarray(apply(x) - b)
    x = np.asarray(x)
    return 0.5 * float(np.dot(r.ravel(), r.ravel())) + 0.5 * lam**2 * float(np.dot(x.ravel(), x.ravel()))


def objective_matrix(op, X, B, lam: float) -> float:
    """Phi_s(X) with the GPU forward operator (solvers.py:144-146)."""
    from .kron import kron_apply

    return objective(lambda Z: kron_apply(op, Z), X, B, lam)


def _norm(a) -> float:
    return float(np.linalg.norm(np.asarray(a).ravel()))


# --------------------------------------------------------------------------------------------
# Lipschitz constant
# --------------------------------------------------------------------------------------------
def _start_vector(seed: int, m: int, n: int, form: str) -> np.ndarray:
    from .rand import stream

    if form == "vector":  # restore(): dims = m*n, F-order un-vec (pipeline.py:117-122,169-171)
        v = stream(seed, "lipschitz").standard_normal((m * n,))
        nv = np.linalg.norm(v.ravel())
        if nv == 0:  # pragma: no cover
            v = np.ones(m * n)
            nv = np.linalg.norm(v)
        v = v / nv
        return v.reshape((m, n), order="F")
    v = stream(seed, "lipschitz").standard_normal((m, n))
    nv = np.linalg.norm(v.ravel())
    if nv == 0:  # pragma: no cover
        v = np.ones((m, n))
        nv = np.linalg.norm(v.ravel())
    return v / nv


def _finish_power(hist: np.ndarray) -> float:
    """Apply solvers.py:123-130 to the device history [iters][2] of (rho, ||w||^2)."""
    rho = 0.0
    for k in range(hist.shape[0]):
        rho = float(hist[k, 0])
        nw2 = float(hist[k, 1])
        if nw2 == 0 or rho <= 0 or not np.isfinite(rho):
            warnings.warn("operator is numerically zero; Lipschitz floor returned")
            return float(np.finfo(float).eps)
    return LIPSCHITZ_SAFETY * rho


def lipschitz(op, iters: int = 50, seed: int = 0, form: str = "matrix", dtype: str = "float64") -> float:
    """estimate_lipschitz on the GPU for a KronOperator: same start vector, iteration count and
    stopping rules as solvers.py:104-130 (matrix form: dims=(m,n); vector form: dims=m*n)."""
    import torch

    from .device import device_operator

    iters = int(iters)
    if iters < 1:
        raise ArgumentError(f"iters must be >= 1, got {iters}")
    m, n = op.shape
    dev = device_operator(op, dtype)
    v0 = _start_vector(seed, m, n, form)
    v = torch.from_numpy(np.ascontiguousarray(v0)).to(dev.device, dev.tdtype)
    hist = dev.power_iter(v, iters)
    return _finish_power(hist[:, :, 0].cpu().numpy())


def make_ops(op, form: str = "matrix", dtype: str = "float64"):
    """(apply, apply_adjoint) closures on the GPU operator, tagged so that ``estimate_lipschitz``
    runs the fused device power iteration instead of a host loop."""
    from .kron import kron_apply, kron_apply_adjoint
    from .psf import unvec, vec

    m, n = op.shape
    if form == "vector":
        def apply(v):
            return vec(kron_apply(op, unvec(v, m, n), dtype=dtype))

        def adjoint(v):
            return vec(kron_apply_adjoint(op, unvec(v, m, n), dtype=dtype))
    else:
        def apply(X):
            return kron_apply(op, X, dtype=dtype)

        def adjoint(X):
            return kron_apply_adjoint(op, X, dtype=dtype)
    apply._kb_power = adjoint._kb_power = (op, form, dtype)
    return apply, adjoint


def estimate_lipschitz(apply, apply_adjoint, dims, iters: int = 50, seed: int = 0) -> float:
    """lambda_max(A^T A) by power iteration, times 1.05 (solvers.py:104-130).

    Closures from ``make_ops`` run on the device (kb_power_iter). Arbitrary host callables keep
    the reference's generic loop — the operator is then whatever the caller computes.
    """
    tag = getattr(apply, "_kb_power", None)
    if tag is not None and getattr(apply_adjoint, "_kb_power", None) is tag:
        op, form, dtype = tag
        want = op.shape[0] * op.shape[1] if form == "vector" else tuple(op.shape)
        got = int(dims) if np.isscalar(dims) else tuple(int(d) for d in dims)
        if got != want:
            raise ArgumentError(f"dims {dims} do not match the operator ({want})")
        return lipschitz(op, iters=iters, seed=seed, form=form, dtype=dtype)
    from .rand import stream

    iters = int(iters)
    if iters < 1:
        raise ArgumentError(f"iters must be >= 1, got {iters}")
    shape = (dims,) if np.isscalar(dims) else tuple(dims)
    v = stream(seed, "lipschitz").standard_normal(shape)
    nv = np.linalg.norm(v.ravel())
    if nv == 0:  # pragma: no cover
        v = np.ones(shape)
        nv = np.linalg.norm(v.ravel())
    v /= nv
    rho = 0.0
    for _ in range(iters):
        w = apply_adjoint(apply(v))
        rho = float(np.vdot(v.ravel(), w.ravel()))
        nw = np.linalg.norm(w.ravel())
        if nw == 0 or rho <= 0:
            warnings.warn("operator is numerically zero; Lipschitz floor returned")
            return float(np.finfo(float).eps)
        v = w / nw
    return LIPSCHITZ_SAFETY * rho


# --------------------------------------------------------------------------------------------
# sFISTA
# --------------------------------------------------------------------------------------------
def _host(t) -> np.ndarray:
    import torch

    return t.to("cpu", torch.float64).numpy().copy()


def sfista(op, B, cfg: SolveConfig, X0=None, truth=None, exact_apply=None, *,
           options: SolveOptions | None = None) -> SolveRun:
    """Accelerated solve of the matrix model against a KronOperator, on the B200."""
    import torch

    from .device import INT_MAX, device_operator, download_pieces, prefault, upload_pieces

    opts = options or SolveOptions()
    fast = not cfg.record_history and not cfg.record_iterates and cfg.rel_tol == 0
    # optional extension: CUDA tensors in skip the host copies on the fast path
    # and x comes back as a float64 CUDA tensor; elsewhere they are brought to the host
    on_device = isinstance(B, torch.Tensor) and B.is_cuda
    if on_device and not fast:
        B, on_device = B.detach().to("cpu", torch.float64).numpy(), False
    if isinstance(X0, torch.Tensor) and not on_device:
        X0 = X0.detach().to("cpu", torch.float64).numpy()
    if not on_device:
        B = np.asarray(B, dtype=float)
    if X0 is not None:  # None: x_0 = 0 (solvers.py:218-219), zeroed on the device
        X0 = X0 if isinstance(X0, torch.Tensor) else np.asarray(X0, dtype=float)
        if X0.shape != B.shape:
            raise ArgumentError(f"x0 shape {X0.shape} does not match data shape {B.shape}")
    if tuple(B.shape) != tuple(op.shape):
        raise ArgumentError(f"image shape {tuple(B.shape)} does not match operator shape {tuple(op.shape)}")
    K = int(cfg.max_iter)
    L, lam = float(cfg.lipschitz), float(cfg.lam)
    ts, beta = momentum_table(K)
    dev = device_operator(op, opts.dtype)
    use_graph = opts.use_graph if opts.use_graph is not None else (fast and K >= 8)

    with dev.exclusive():
        stream = torch.cuda.current_stream()
        hB, hX = dev.staging("host_b", pinned=True), dev.staging("host_x", pinned=True)
        Bd, Xd, Yd = dev.staging("b"), dev.staging("x"), dev.staging("y")
        if on_device:
            Bd.copy_(B)
        else:
            upload_pieces(Bd, B, hB)
        if X0 is None:
            Xd.zero_()
        elif isinstance(X0, torch.Tensor):
            Xd.copy_(X0)
        else:
            upload_pieces(Xd, X0, hX)
        Yd.copy_(Xd)
        flag = torch.full((1,), INT_MAX, dtype=torch.int32, device=dev.device)
        start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

        if fast:
            start.record(stream)
            dev.sfista_run(Bd, Xd, Yd, beta, 0, K, L, lam, opts.project, flag, use_graph=use_graph)
            stop.record(stream)
            if on_device:
                x = Xd.to(torch.float64, copy=True)
            else:  # the result array's pages are first touched while the GPU iterates
                out = np.empty(B.shape)
                x = download_pieces(Xd, hX, out, after=prefault(out))
            torch.cuda.current_stream().synchronize()
            bad = int(flag.item())
            if bad <= K:
                raise NumericError(f"non-finite iterate at iteration {bad}")
            return SolveRun(x=x, iterations=K, solve_ms=float(start.elapsed_time(stop)))

        # History / iterate / rel_tol path, one native iteration per step. Per iteration k the
        # device holds hist[k-1] = (||x_k - x_{k-1}||^2, ||x_{k-1}||^2, ||x_k||^2, -, from the
        # update epilogue; ||A x_k - b||^2, ||x_k - truth||^2 from one extra forward application
        # plus kb_resid_norms). Nothing comes back to the host per iteration unless a host-side
        # quantity needs it (rel_tol stopping, record_iterates, a host exact_apply callable);
        # otherwise one synchronisation at the end. solve_ms / ms time only the iteration's own
        # kernels (solvers.py:169-174), bracketed by events on the stream.
        norm_b = _norm(B)
        norm_truth = _norm(truth) if truth is not None else 0.0
        hist = torch.zeros((K, 8), dtype=torch.float64, device=dev.device)
        truth_d = None
        if cfg.record_history and truth is not None:
            truth_d = torch.from_numpy(np.ascontiguousarray(truth, dtype=np.float64)).to(dev.device, dev.tdtype)
        Ax = dev.staging("ax") if cfg.record_history else None
        per_iter_host = cfg.rel_tol > 0 or cfg.record_iterates or (cfg.record_history and exact_apply is not None)
        marks = []
        gammas, iterates = [], []
        iterations = 0
        for k in range(1, K + 1):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            dev.sfista_run(Bd, Xd, Yd, beta, k - 1, 1, L, lam, opts.project, flag, norms=hist[k - 1, :4],
                           use_graph=False)
            e1.record(stream)
            marks.append((e0, e1))
            if cfg.record_history:
                dev.apply(Xd, out=Ax)
                dev.resid_norms(Ax, Bd, Xd, truth_d, hist[k - 1, 4:6])
            iterations = k
            if not per_iter_host:
                continue
            e1.synchronize()
            if int(flag.item()) <= k:
                raise NumericError(f"non-finite iterate at iteration {k}")
            if cfg.record_iterates or (cfg.record_history and exact_apply is not None):
                x = _host(Xd)
                if cfg.record_iterates:
                    iterates.append(x.copy())
                if cfg.record_history and exact_apply is not None:
                    gammas.append(_norm(exact_apply(x) - B) / norm_b if norm_b > 0 else None)
            if cfg.rel_tol > 0:
                step, base = np.sqrt(hist[k - 1, :2].cpu().numpy())
                if step < cfg.rel_tol * (base if base > 0 else 1.0):
                    break
        torch.cuda.current_stream().synchronize()
        bad = int(flag.item())
        if bad <= iterations:
            raise NumericError(f"non-finite iterate at iteration {bad}")
        h = hist[:iterations].cpu().numpy()
        elapsed, history = 0.0, []
        for k in range(1, iterations + 1):
            elapsed += float(marks[k - 1][0].elapsed_time(marks[k - 1][1]))
            if cfg.record_history:
                r2, x2, e2 = h[k - 1, 4], h[k - 1, 2], h[k - 1, 5]
                phi = 0.5 * float(r2) + 0.5 * lam**2 * float(x2)
                eta = float(np.sqrt(e2)) / norm_truth if truth is not None and norm_truth > 0 else None
                gamma = gammas[k - 1] if exact_apply is not None else None
                history.append(IterationRecord(k=k, t=float(ts[k - 1]), objective=phi, eta=eta,
                                               gamma=gamma, ms=elapsed))
        return SolveRun(x=_host(Xd), iterations=iterations, solve_ms=elapsed, history=history,
                        iterates=iterates)


LAMBDA_DENSE_LIMIT = 1024  # solvers.py:47
LAMBDA_PROBE_TERMS = 5     # solvers.py:50


def select_lambda(op, B, noise_level: float, lipschitz: float, grid_points: int = 25,
                  probe_iters: int = 50) -> float:
    """Discrepancy-principle lambda over the reference's log grid (solvers.py:255-306).

    Same validation, grid, target and argmin. Small problems (m n <= LAMBDA_DENSE_LIMIT) take the
    reference's dense eigendecomposition route unchanged (host setup on <= 1024 unknowns). Larger
    ones run the fixed sFISTA probes — 25 independent 50-iteration solves on the truncated
    operator, one per candidate lambda — as ONE batched device solve (one image per lambda,
    kb_sfista_run_lams; the batched cfg3 kernels), then one batched forward application and the
    per-image residual norms on the device, instead of 25 sequential solves."""
    from .kron import kron_to_dense
    from .psf import vec

    B = np.asarray(B, dtype=float)
    if B.shape != tuple(op.shape):
        raise ArgumentError(f"data shape {B.shape} does not match operator shape {tuple(op.shape)}")
    if not (np.isfinite(noise_level) and noise_level >= 0):
        raise ArgumentError(f"noise level must be >= 0, got {noise_level}")
    if not (np.isfinite(lipschitz) and lipschitz > 0):
        raise ArgumentError(f"Lipschitz constant must be positive, got {lipschitz}")
    scale = np.sqrt(lipschitz)
    grid = np.geomspace(1e-4 * scale, scale, int(grid_points))
    b = vec(B)
    target = noise_level * np.linalg.norm(b)
    m, n = op.shape
    if m * n <= LAMBDA_DENSE_LIMIT:
        A = kron_to_dense(op)
        w, Q = np.linalg.eigh(A.T @ A)
        z = Q.T @ (A.T @ b)
        bb = float(b @ b)
        residuals = np.empty(grid.size)
        for i, lam in enumerate(grid):
            xh = z / (w + lam**2)
            residuals[i] = np.sqrt(max(bb - 2.0 * float(z @ xh) + float((w * xh) @ xh), 0.0))
        return float(grid[int(np.argmin(np.abs(residuals - target)))])
    residuals = lambda_probe_residuals(op.truncate(min(LAMBDA_PROBE_TERMS, len(op.terms))), B, grid,
                                       lipschitz, int(probe_iters))
    return float(grid[int(np.argmin(np.abs(residuals - target)))])


def lambda_probe_residuals(probe, B, grid, lipschitz: float, iters: int) -> np.ndarray:
    """||A_s x(lam) - B||_F of the 50-iteration sFISTA probe from X0 = 0 for every lam of the grid
    (solvers.py:296-305), batched over the grid on the device (chunked to the free memory)."""
    import torch

    from .device import INT_MAX, DeviceOperator

    m, n = probe.shape
    _, beta = momentum_table(int(iters))
    free = torch.cuda.mem_get_info()[0]
    per_image = (len(probe.terms) + 8) * m * n * 8  # Z planes + halo, R, B, X, Y, AX (fp64)
    chunk = int(max(1, min(len(grid), (free // 2) // per_image)))
    out = np.empty(len(grid))
    for c0 in range(0, len(grid), chunk):
        lams = np.asarray(grid[c0:c0 + chunk], dtype=np.float64)
        G = lams.size
        dev = DeviceOperator([probe] * G, "float64")
        Bd = torch.from_numpy(np.ascontiguousarray(B)).to(dev.device).expand(G, m, n).contiguous()
        Xd = torch.zeros_like(Bd)
        Yd = torch.zeros_like(Bd)
        flag = torch.full((1,), INT_MAX, dtype=torch.int32, device=dev.device)
        dev.sfista_run(Bd, Xd, Yd, beta, 0, int(iters), lipschitz, lams, False, flag, use_graph=False)
        AX = dev.apply(Xd)
        r2 = dev.resid_norms_images(AX, Bd)
        bad = int(flag.item())
        if bad <= iters:
            raise NumericError(f"non-finite iterate at iteration {bad}")
        out[c0:c0 + G] = np.sqrt(r2)
    return out


def sfista_batch(ops, B, lipschitz, lam: float, iters: int, *, options: SolveOptions | None = None,
                 X0=None):
    """Batch of independent solves (BASELINE cfg3): one batched operator, per-image L, shared lam
    and momentum. B: (batch, m, n) numpy or CUDA tensor. Returns (x, solve_ms) with x like B."""
    import torch

    from .device import INT_MAX, DeviceOperator, download_pieces, prefault, upload_pieces

    opts = options or SolveOptions()
    dev = ops if isinstance(ops, DeviceOperator) else DeviceOperator(list(ops), opts.dtype)
    _, beta = momentum_table(int(iters))
    on_device = isinstance(B, torch.Tensor) and B.is_cuda
    if on_device:
        Bd = B.to(dev.tdtype).contiguous()
    else:  # host arrays move in pinned pieces (device.upload_pieces), converted on the way
        Bd = dev.staging("b")
        upload_pieces(Bd, np.asarray(B), dev.staging("host_b", pinned=True))
    if X0 is None:
        Xd = torch.zeros_like(Bd)
    else:
        Xd = (X0 if isinstance(X0, torch.Tensor) else torch.from_numpy(np.asarray(X0))).to(dev.device, dev.tdtype).contiguous()
    Yd = Xd.clone()
    flag = torch.full((1,), INT_MAX, dtype=torch.int32, device=dev.device)
    stream = torch.cuda.current_stream()
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    start.record(stream)
    dev.sfista_run(Bd, Xd, Yd, beta, 0, int(iters), lipschitz, lam, opts.project, flag,
                   use_graph=bool(opts.use_graph))
    stop.record(stream)
    out, touched = None, ()
    if not on_device:  # the result array's pages are first touched while the GPU iterates
        out = np.empty(tuple(Xd.shape))
        touched = prefault(out)
    stop.synchronize()
    bad = int(flag.item())
    if bad <= iters:
        raise NumericError(f"non-finite iterate at iteration {bad}")
    x = Xd if on_device else download_pieces(Xd, dev.staging("host_x", pinned=True), out, after=touched)
    return x, float(start.elapsed_time(stop))
