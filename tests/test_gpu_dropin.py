"""The zero-edit drop-in on the GPU: the reference's own callers run through ``install()``.

The unmodified reference package (pip-installed into baseline/_ref by __graft_entry__.build(),
test-only) is called twice on identical inputs: once as shipped (its CPU numpy path) and once
after ``kb.install(kronblur)`` rerouted every by-name binding to the device. ``restore()``
(pipeline.py:143-227) then runs our support-block ``decompose``, the vector-form Lipschitz
estimate on ``kb_power_iter`` (pipeline.py:169-171), our ``select_lambda`` probes when lam is None
(solvers.py:294-305), the device sFISTA with history and the device ``blur_direct`` as its
``exact_apply``. Everything the result reports must agree with the reference's own run.
"""

import numpy as np
import pytest

from conftest import cuda_ok, reference_module

import paper_1901_00913_b200 as kb

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_ok(), reason="needs a CUDA device")]


def _problem(kronblur, m, n, seed):
    from kronblur import psf as rpsf

    rng = np.random.default_rng(seed)
    X = np.zeros((m, n))
    for _ in range(12):
        r0, c0 = rng.integers(0, m - 8), rng.integers(0, n - 8)
        X[r0:r0 + rng.integers(4, 20), c0:c0 + rng.integers(4, 20)] = rng.random()
    y, x = np.mgrid[-4:5, -4:5]
    g = np.exp(-0.5 * ((x / 2.2) ** 2 + (y / 1.3) ** 2 + 0.4 * x * y))
    psf = rpsf.Psf(g / g.sum(), (5, 5))
    return X, psf, rng


@pytest.mark.parametrize("bc_name", ["zero", "reflective"])
def test_restore_through_install_matches_the_reference(bc_name):
    kronblur = reference_module()
    if kronblur is None:
        pytest.skip("reference not installed in baseline/_ref")
    from kronblur import pipeline, psf as rpsf

    bc = rpsf.BoundaryCondition(bc_name)
    X, psf, rng = _problem(kronblur, 96, 96, 3)
    b = rpsf.blur_direct(rpsf.pad_to(psf, 96, 96), X, bc)
    B = b + 0.01 * np.linalg.norm(b) / np.sqrt(b.size) * rng.standard_normal(b.shape)
    args = dict(method="sfista", s=3, lam=0.03, iters=40, truth=X, seed=2)
    ref = pipeline.restore(B, psf, bc, **args)  # the reference, CPU, as shipped
    undo = kb.install(kronblur)
    try:
        got = pipeline.restore(B, psf, bc, **args)
    finally:
        undo()
    assert (got.s, got.rank, got.iterations) == (ref.s, ref.rank, ref.iterations)
    assert got.eps == pytest.approx(ref.eps, rel=1e-9, abs=1e-14)
    # vector-form power iteration (F-order start) on the full-rank operator: same sequence
    assert got.lipschitz == pytest.approx(ref.lipschitz, rel=1e-10)
    err = np.linalg.norm(got.restored - ref.restored) / np.linalg.norm(ref.restored)
    assert err <= 1e-9, f"restored image differs: {err:.3e}"
    assert got.gamma == pytest.approx(ref.gamma, rel=1e-9)
    assert got.eta == pytest.approx(ref.eta, rel=1e-9)
    assert len(got.history) == len(ref.history) == 40
    for h, r in zip(got.history, ref.history):
        assert (h.k, h.t) == (r.k, r.t)
        assert h.objective == pytest.approx(r.objective, rel=1e-9)
        assert h.eta == pytest.approx(r.eta, rel=1e-8)
        assert h.gamma == pytest.approx(r.gamma, rel=1e-8)
    assert isinstance(got.history[0], kronblur.solvers.IterationRecord)


def test_restore_with_automatic_lambda_through_install():
    """lam=None: the discrepancy principle over the 25-point grid (solvers.py:255-306) picks the
    same lambda through the batched device probes as the reference's sequential CPU probes."""
    kronblur = reference_module()
    if kronblur is None:
        pytest.skip("reference not installed in baseline/_ref")
    from kronblur import pipeline, psf as rpsf

    bc = rpsf.BoundaryCondition.ZERO
    X, psf, rng = _problem(kronblur, 48, 48, 7)  # m*n > 1024: the probe route
    b = rpsf.blur_direct(rpsf.pad_to(psf, 48, 48), X, bc)
    B = b + 0.02 * np.linalg.norm(b) / np.sqrt(b.size) * rng.standard_normal(b.shape)
    args = dict(method="sfista", s=2, lam=None, noise_level=0.02, iters=20, truth=X, record_history=False)
    ref = pipeline.restore(B, psf, bc, **args)
    undo = kb.install(kronblur)
    try:
        got = pipeline.restore(B, psf, bc, **args)
    finally:
        undo()
    # same grid point; the grid scales with sqrt(L), whose last bits differ (device power iteration)
    assert got.lambda_used == pytest.approx(ref.lambda_used, rel=1e-12)
    err = np.linalg.norm(got.restored - ref.restored) / np.linalg.norm(ref.restored)
    assert err <= 1e-9


def test_install_options_reach_the_solver():
    """kb.install(kronblur, options=...) applies the options to every patched sfista call: with
    projection on, the result is the projected solve (x >= 0), in float32 within 1e-4 of fp64."""
    kronblur = reference_module()
    if kronblur is None:
        pytest.skip("reference not installed in baseline/_ref")
    from kronblur import kron, psf as rpsf, solvers

    bc = rpsf.BoundaryCondition.REFLECTIVE
    X, psf, rng = _problem(kronblur, 64, 64, 11)
    op = kron.decompose(rpsf.pad_to(psf, 64, 64), bc, s=3)
    B = kron.kron_apply(op, X) + 0.01 * rng.standard_normal((64, 64))
    cfg = solvers.SolveConfig(lam=0.05, lipschitz=1.2, max_iter=30, record_history=False)
    plain = solvers.sfista(op, B, cfg).x
    undo = kb.install(kronblur, options=kb.SolveOptions(dtype="float64", project=True))
    try:
        proj64 = solvers.sfista(op, B, cfg).x
    finally:
        undo()
    undo = kb.install(kronblur, options=kb.SolveOptions(dtype="float32", project=True))
    try:
        proj32 = solvers.sfista(op, B, cfg).x
    finally:
        undo()
    assert plain.min() < 0 and proj64.min() >= 0
    assert np.linalg.norm(proj32 - proj64) / np.linalg.norm(proj64) <= 1e-4
