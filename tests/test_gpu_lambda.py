"""select_lambda (solvers.py:255-306) on the device: the probe route's 25 candidate solves run as
one batched sFISTA solve (kb_sfista_run_lams). Checked against the reference's golden choices and
the oracle's probe residuals (fp64, 1e-10 relative)."""

import os

import numpy as np
import pytest

from conftest import GOLDEN, cuda_ok

pytestmark = pytest.mark.gpu

if not cuda_ok():  # pragma: no cover - collected on CPU but skipped
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1901_00913_b200 as kb  # noqa: E402
from paper_1901_00913_b200.solvers import LAMBDA_PROBE_TERMS, lambda_probe_residuals  # noqa: E402
from oracle import kronblur_port as port  # noqa: E402


def cases():
    g = np.load(os.path.join(GOLDEN, "lambda.npz"))
    for ci in range(int(g["ncases"])):
        psf = kb.Psf(g[f"l{ci}_psf"], tuple(int(v) for v in g[f"l{ci}_center"]))
        B = g[f"l{ci}_B"]
        noise, L = (float(v) for v in g[f"l{ci}_noise_L"])
        op = kb.decompose(psf, kb.BoundaryCondition(str(g[f"l{ci}_bc"])), shape=B.shape)
        yield op, B, noise, L, float(g[f"l{ci}_lam"])


def test_select_lambda_matches_reference_choices():
    for op, B, noise, L, want in cases():
        assert kb.select_lambda(op, B, noise, L) == want


def test_probe_residuals_match_oracle():
    for op, B, noise, L, _ in cases():
        if B.size <= 1024:
            continue
        _, want = port.select_lambda(op, B, noise, L)
        grid = np.geomspace(1e-4 * np.sqrt(L), np.sqrt(L), 25)
        probe = op.truncate(min(LAMBDA_PROBE_TERMS, len(op.terms)))
        got = lambda_probe_residuals(probe, B, grid, L, 50)
        np.testing.assert_allclose(got, want, rtol=1e-10, atol=0)


def test_select_lambda_validation():
    op, B, noise, L, _ = next(iter(cases()))
    with pytest.raises(kb.ArgumentError):
        kb.select_lambda(op, B, -1.0, L)
    with pytest.raises(kb.ArgumentError):
        kb.select_lambda(op, B, noise, 0.0)
    with pytest.raises(kb.ArgumentError):
        kb.select_lambda(op, B[:-1], noise, L)
