"""record_history / rel_tol / record_iterates path of sfista (solvers.py:176-197) against the
oracle: objective (solvers.py:133-141) from the device residual norms, eta against a truth image,
gamma through an exact_apply callable (here the oracle's blur_direct, psf.py:170-193), t_k, the
cumulative ms, and the rel_tol stopping iteration. Tolerance fp64 1e-12 relative on the scalars
(they differ from the reference only by summation order); fp32 1e-4."""

import numpy as np
import pytest

from conftest import cuda_ok, random_psf

pytestmark = pytest.mark.gpu

if not cuda_ok():  # pragma: no cover - collected on CPU but skipped
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1901_00913_b200 as kb  # noqa: E402
from oracle import kronblur_port as port  # noqa: E402


def oracle_history(op, psf, bc, B, truth, L, lam, iters):
    _, its = port.sfista(op, B, L, lam, iters, record_iterates=True)
    pop = port.PortOperator(op)
    out = []
    for x in its:
        r = port.kron_apply(pop, x) - B
        phi = 0.5 * float(r.ravel() @ r.ravel()) + 0.5 * lam**2 * float(x.ravel() @ x.ravel())
        eta = np.linalg.norm(x - truth) / np.linalg.norm(truth)
        gamma = np.linalg.norm(port.blur_direct(psf.values, psf.center, x, bc) - B) / np.linalg.norm(B)
        out.append((phi, eta, gamma))
    return its, out


@pytest.mark.parametrize("dtype,tol", [("float64", 1e-12), ("float32", 1e-4)])
@pytest.mark.parametrize("bc", [kb.BoundaryCondition.ZERO, kb.BoundaryCondition.REFLECTIVE])
def test_history_matches_oracle(rng, dtype, tol, bc):
    psf = random_psf(rng, 7)
    m = 64
    op = kb.decompose(psf, bc, s=3, shape=(m, m))
    truth = rng.random((m, m))
    B = kb.kron_apply(op, truth) + 0.01 * rng.standard_normal((m, m))
    L, lam, iters = 1.3, 0.05, 25
    its, want = oracle_history(op, psf, bc.value, B, truth, L, lam, iters)
    exact = lambda x: port.blur_direct(psf.values, psf.center, x, bc.value)  # noqa: E731
    cfg = kb.SolveConfig(lam=lam, lipschitz=L, max_iter=iters, record_history=True)
    run = kb.sfista(op, B, cfg, truth=truth, exact_apply=exact, options=kb.SolveOptions(dtype=dtype))
    assert run.iterations == iters and len(run.history) == iters
    for k, (h, (phi, eta, gamma)) in enumerate(zip(run.history, want), start=1):
        assert h.k == k
        assert abs(h.objective - phi) <= tol * abs(phi), (k, h.objective, phi)
        assert abs(h.eta - eta) <= tol * eta
        assert abs(h.gamma - gamma) <= tol * gamma
    ms = [h.ms for h in run.history]
    assert all(b >= a for a, b in zip(ms, ms[1:])) and abs(ms[-1] - run.solve_ms) < 1e-9
    t = 1.0
    for h in run.history:  # t_k recorded before the update (solvers.py:186)
        assert h.t == t
        t = port.momentum_next(t)
    rel = np.linalg.norm(run.x - its[-1]) / np.linalg.norm(its[-1])
    assert rel <= (1e-12 if dtype == "float64" else 1e-4)


def test_history_without_truth_or_exact_apply(rng):
    psf = random_psf(rng, 5)
    op = kb.decompose(psf, kb.BoundaryCondition.ZERO, s=2, shape=(40, 40))
    B = rng.random((40, 40))
    run = kb.sfista(op, B, kb.SolveConfig(lam=0.1, lipschitz=1.2, max_iter=10))
    assert len(run.history) == 10
    assert all(h.eta is None and h.gamma is None for h in run.history)
    _, its = port.sfista(op, B, 1.2, 0.1, 10, record_iterates=True)
    r = port.kron_apply(port.PortOperator(op), its[-1]) - B
    phi = 0.5 * float(r.ravel() @ r.ravel()) + 0.5 * 0.01 * float(its[-1].ravel() @ its[-1].ravel())
    assert abs(run.history[-1].objective - phi) <= 1e-12 * phi


def test_rel_tol_stops_at_the_oracle_iteration(rng):
    psf = random_psf(rng, 5)
    op = kb.decompose(psf, kb.BoundaryCondition.REFLECTIVE, s=3, shape=(48, 48))
    B = rng.random((48, 48))
    pop = port.PortOperator(op)
    L = port.estimate_lipschitz(lambda v: port.kron_apply(pop, v), lambda v: port.kron_apply_adjoint(pop, v),
                                (48, 48), 50, 0)
    lam, tol_rel = 0.2, 1e-2
    _, its = port.sfista(op, B, L, lam, 300, record_iterates=True)
    prev = np.zeros_like(B)
    stop = None
    for k, x in enumerate(its, start=1):  # solvers.py:178-179, 197
        step, base = np.linalg.norm(x - prev), np.linalg.norm(prev)
        if step < tol_rel * (base if base > 0 else 1.0):
            stop = k
            break
        prev = x
    assert stop is not None and stop < 300
    run = kb.sfista(op, B, kb.SolveConfig(lam=lam, lipschitz=L, max_iter=300, rel_tol=tol_rel,
                                          record_history=False))
    assert run.iterations == stop
    assert np.max(np.abs(run.x - its[stop - 1])) <= 1e-12 * np.max(np.abs(its[stop - 1]))
