"""Property tests restated from the reference suite with the B200 solver substituted:
* the global O(1/k^2) rate bound of FISTA (kronblur tests/test_solvers.py:173-191) on a Kronecker
  operator, against the dense Tikhonov optimum;
* bitwise determinism of repeated runs, history included (test_solvers.py:341-351), on the fp64
  DMMA, fp32 mma.sync and fp32 tcgen05 paths;
* the untruncated operator equals the direct blur (acceptance criterion 2,
  test_acceptance.py:111-131, 1e-8), here with both sides on the device."""

import numpy as np
import pytest

from conftest import cuda_ok, random_psf

pytestmark = pytest.mark.gpu

if not cuda_ok():  # pragma: no cover - collected on CPU but skipped
    pytest.skip("needs a CUDA device", allow_module_level=True)

import torch  # noqa: E402

import paper_1901_00913_b200 as kb  # noqa: E402
from oracle import kronblur_port as port  # noqa: E402


@pytest.mark.parametrize("bc", [kb.BoundaryCondition.ZERO, kb.BoundaryCondition.REFLECTIVE])
def test_rate_bound_against_tikhonov_optimum(rng, bc):
    m = 12
    psf = random_psf(rng, 5)
    op = kb.decompose(psf, bc, shape=(m, m))
    Ad = np.zeros((m * m, m * m))
    for t in op.terms:  # A = sum_i K_i (x) H_i acting on vec (column-major) images
        Ad += np.kron(port.dense_factor(t.K), port.dense_factor(t.H))
    B = rng.standard_normal((m, m))
    b = B.flatten(order="F")
    lam = 0.4
    L = kb.lipschitz(op, iters=200, seed=0)
    xstar = np.linalg.solve(Ad.T @ Ad + lam**2 * np.eye(m * m), Ad.T @ b)

    def phi(x):
        r = Ad @ x - b
        return 0.5 * float(r @ r) + 0.5 * lam**2 * float(x @ x)

    phistar = phi(xstar)
    run = kb.sfista(op, B, kb.SolveConfig(lam=lam, lipschitz=L, max_iter=100, record_iterates=True))
    c = 2.0 * (L + lam**2) * float(xstar @ xstar)
    assert len(run.iterates) == run.iterations == 100
    for k, xk in enumerate(run.iterates, start=1):
        assert phi(xk.flatten(order="F")) - phistar <= c / (k + 1) ** 2 + 1e-12, k


@pytest.mark.parametrize("dtype,m,w", [("float64", 96, 9), ("float32", 96, 9), ("float32", 1024, 65)])
def test_runs_are_bitwise_deterministic(rng, dtype, m, w):
    vals = np.outer(np.hanning(w + 2)[1:-1], np.hanning(w + 2)[1:-1]) + 0.01 * rng.random((w, w))
    psf = kb.Psf(vals / vals.sum(), ((w + 1) // 2, (w + 1) // 2))
    op = kb.decompose(psf, kb.BoundaryCondition.ZERO, s=2, shape=(m, m))
    B = rng.random((m, m))
    cfg = kb.SolveConfig(lam=0.05, lipschitz=1.0, max_iter=12, record_history=True)
    opts = kb.SolveOptions(dtype=dtype, project=True)
    r1 = kb.sfista(op, B, cfg, options=opts)
    r2 = kb.sfista(op, B, cfg, options=opts)
    assert np.array_equal(r1.x, r2.x)
    assert [h.objective for h in r1.history] == [h.objective for h in r2.history]


@pytest.mark.parametrize("bc", [kb.BoundaryCondition.ZERO, kb.BoundaryCondition.REFLECTIVE])
def test_untruncated_operator_is_the_direct_blur(rng, bc):
    m = 64
    psf = kb.pad_to(random_psf(rng, 9), m, m)
    op = kb.decompose(psf, bc, shape=(m, m))  # full rank
    X = torch.from_numpy(rng.random((m, m))).cuda()
    from paper_1901_00913_b200.device import device_operator

    AX = device_operator(op, "float64").apply(X)
    blur = kb.blur_direct(psf, X, bc)
    assert float(torch.linalg.norm(AX - blur) / torch.linalg.norm(blur)) <= 1e-8
