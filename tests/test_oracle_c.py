"""Pin the C restatement (oracle/kb_oracle.c) to the reference before trusting it at full size.

* against the reference's own outputs (tests/golden/, made by running kronblur itself):
  kron_apply / kron_apply_adjoint on reference-built operators, the matrix-form Lipschitz
  estimate, projected solves, the cfg1 solution at full size, and blur_direct bit for bit;
* bit-exact on integer data against the dense index rules (structured.py:111-123), both
  boundary conditions, forward and adjoint;
* against the numpy port (oracle/kronblur_port.py) on random operators.
No GPU is needed.
"""

import os

import numpy as np
import pytest

from conftest import GOLDEN

import paper_1901_00913_b200 as kb
from oracle import kb_oracle as C
from oracle import kronblur_port as port


class Fac:
    def __init__(self, kind, c, j):
        self.kind, self.c, self.j, self.n = kind, np.asarray(c, float), int(j), len(c)


class Term:
    def __init__(self, H, K):
        self.H, self.K = H, K


class Op:
    def __init__(self, terms, shape):
        self.terms, self.shape = tuple(terms), tuple(shape)


def golden_op(g, pre):
    kind = str(g[pre + "kind"])
    Hc, Kc = g[pre + "H_c"], g[pre + "K_c"]
    m = Hc.shape[1]
    return Op([Term(Fac(kind, Hc[i], g[pre + "H_j"]), Fac(kind, Kc[i], g[pre + "K_j"])) for i in range(Hc.shape[0])],
              (m, Kc.shape[1]))


def test_apply_matches_reference_golden():
    g = np.load(os.path.join(GOLDEN, "kron_small.npz"))
    for c in range(6):
        pre = f"c{c}_"
        op = golden_op(g, pre)
        oop = C.OracleOp(op)
        X = g[pre + "X"]
        for got, want in ((C.apply(oop, X), g[pre + "AX"]), (C.apply(oop, X, adjoint=True), g[pre + "AtX"])):
            err = np.linalg.norm(got - want) / np.linalg.norm(want)
            assert err <= 1e-12, (c, err)


def test_power_iteration_and_projected_solve_match_reference_golden():
    g = np.load(os.path.join(GOLDEN, "kron_small.npz"))
    for c in range(6):
        pre = f"c{c}_"
        op = golden_op(g, pre)
        oop = C.OracleOp(op)
        m, n = op.shape
        rho, nw2 = C.power(oop, port.lipschitz_start(c, (m, n)), 50)
        assert 1.05 * rho[-1] == pytest.approx(float(g[pre + "L_mat"]), rel=1e-11)
        L = float(g[pre + "L_mat"])
        _, beta = kb.momentum_table(40)
        x = C.sfista(oop, g[pre + "B"], L, 0.05, 40, beta, project=True)
        want = g[pre + "x_proj"]
        assert np.linalg.norm(x - want) / np.linalg.norm(want) <= 1e-10


def test_cfg1_full_size_solution_matches_reference():
    """BASELINE cfg1 (256^2, zero BC, w=31, r=3, 100 projected iterations) with the reference's
    own factors, data and L: the C oracle reproduces the reference's projected solution."""
    g = np.load(os.path.join(GOLDEN, "cfg1.npz"))
    op = golden_op(g, "")
    _, beta = kb.momentum_table(100)
    x = C.sfista(C.OracleOp(op), g["B"], float(g["L"]), 0.02, 100, beta, project=True)
    err = np.linalg.norm(x - g["x_proj"]) / np.linalg.norm(g["x_proj"])
    assert err <= 1e-11, err
    # unprojected: the reference's own sfista
    x0 = C.sfista(C.OracleOp(op), g["B"], float(g["L"]), 0.02, 100, beta, project=False)
    assert np.linalg.norm(x0 - g["x_sfista"]) / np.linalg.norm(g["x_sfista"]) <= 1e-11


@pytest.mark.parametrize("kind", ["toeplitz", "toeplitz_plus_hankel"])
@pytest.mark.parametrize("shape", [(17, 23), (32, 32), (5, 40), (64, 9)])
def test_integer_data_bit_exact_against_dense_rules(kind, shape):
    rng = np.random.default_rng(hash((kind, shape)) % 2**32)
    m, n = shape
    terms = []
    for _ in range(3):
        ha, hb = min(6, m - 1), min(5, n - 1)
        ca, cb = np.zeros(m), np.zeros(n)
        ja, jb = int(rng.integers(1, m + 1)), int(rng.integers(1, n + 1))
        for d in range(-ha, ha + 1):
            if 1 <= ja + d <= m:
                ca[ja + d - 1] = rng.integers(-5, 6)
        for d in range(-hb, hb + 1):
            if 1 <= jb + d <= n:
                cb[jb + d - 1] = rng.integers(-5, 6)
        terms.append(Term(Fac(kind, ca, ja), Fac(kind, cb, jb)))
    op = Op(terms, shape)
    X = rng.integers(-9, 10, size=shape).astype(float)
    oop = C.OracleOp(op, rel_tol=0.0)
    assert np.array_equal(C.apply(oop, X), port.dense_kron_apply(op, X))
    assert np.array_equal(C.apply(oop, X, adjoint=True), port.dense_kron_apply(op, X, adjoint=True))


@pytest.mark.parametrize("bc", ["zero", "reflective"])
def test_random_operator_matches_numpy_port(bc):
    rng = np.random.default_rng(3 if bc == "zero" else 4)
    vals = rng.random((11, 9)) + 0.05
    psf = kb.Psf(vals / vals.sum(), (6, 4))
    op = kb.decompose(psf, kb.BoundaryCondition(bc), s=4, shape=(96, 96))
    oop, pop = C.OracleOp(op), port.PortOperator(op)
    X = rng.standard_normal((96, 96))
    for adj in (False, True):
        got = C.apply(oop, X, adj)
        want = (port.kron_apply_adjoint if adj else port.kron_apply)(pop, X)
        assert np.linalg.norm(got - want) / np.linalg.norm(want) <= 1e-12
    B = port.kron_apply(pop, X) + 0.01 * rng.standard_normal((96, 96))
    _, beta = kb.momentum_table(30)
    want, _ = port.sfista(op, B, 1.1, 0.03, 30, project=True)
    got = C.sfista(oop, B, 1.1, 0.03, 30, beta, project=True)
    assert np.linalg.norm(got - want) / np.linalg.norm(want) <= 1e-12


def test_blur_direct_bit_identical_to_reference_golden():
    g = np.load(os.path.join(GOLDEN, "blur.npz"))
    for c in range(int(g["ncases"])):
        pre = f"b{c}_"
        for bc in ("zero", "reflective"):
            got = C.blur_direct(g[pre + "psf"], g[pre + "center"], g[pre + "X"], bc)
            assert np.array_equal(got, g[pre + f"{bc}_Y"]), (c, bc)


def test_projection_keeps_nan_and_maps_negative_zero():
    """np.maximum(x, 0) semantics: the non-finite check must still see NaN."""
    op = Op([Term(Fac("toeplitz", [0, 1, 0], 2), Fac("toeplitz", [0, 1, 0], 2))], (3, 3))
    B = np.full((3, 3), np.nan)
    with pytest.raises(FloatingPointError, match="iteration 1"):
        C.sfista(C.OracleOp(op, rel_tol=0.0), B, 1.0, 0.5, 3, np.zeros(3), project=True)
