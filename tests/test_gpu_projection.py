"""The x >= 0 projection and the boundary index logic, bit-exact on exact inputs (SURVEY §7 step 4,
F3, F5): with integer generators, integer data and X0, L = 0.75 and lam = 0.5 (so L + lam^2 = 1),
the first sFISTA iteration is exact in both dtypes: x_1 = max(0.75 y_0 - A^T(A y_0 - b), 0) is a
multiple of 1/4 far below 2^22, and every 3xTF32 operand is an integer of <= 11 bits (exact in the
tf32 hi part). In fp64 the second is exact too: beta_1 = (t_1 - 1)/t_2 = 0 so y_2 = x_1, and x_2
is a multiple of 1/16 far below 2^53 (in fp32 its partial sums outgrow 24 bits). The
device result (fp64 DMMA, fp32 3xTF32 on mma.sync or tcgen05 by the default policy) must then be
bit-identical to the C oracle (oracle/kb_oracle.c), the clamp mask included, for both boundary
conditions.
"""

import numpy as np
import pytest

from conftest import cuda_ok

pytestmark = pytest.mark.gpu

if not cuda_ok():  # pragma: no cover - collected on CPU but skipped
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1901_00913_b200 as kb  # noqa: E402
from oracle import kb_oracle as C  # noqa: E402
from paper_1901_00913_b200.device import device_operator  # noqa: E402


def sparse_int_operator(rng, m, n, r, bc, h, nnz=5):
    """Integer generators with `nnz` nonzero taps (values in +-1, +-2) spread over a band of
    half width h: wide bands (tensor-core passes) with small exact partial sums."""
    make = kb.toep if bc == "zero" else kb.toep_plus_hank
    ja, jb = m // 2 + 1, n // 2 + 1
    terms = []
    for _ in range(r):
        a, b = np.zeros(m), np.zeros(n)
        for c, j in ((a, ja), (b, jb)):
            offs = rng.choice(np.arange(-h, h + 1), size=nnz, replace=False)
            offs[0], offs[1] = -h, h  # the full band width is present
            c[j - 1 + offs] = rng.choice([-2.0, -1.0, 1.0, 2.0], size=nnz)
        terms.append(kb.KronTerm(sigma=1.0, H=make(a, ja), K=make(b, jb)))
    return kb.KronOperator(terms=tuple(terms), shape=(m, n), bc=kb.BoundaryCondition(bc),
                           sigma=np.ones(r), s=r, rank=r, eps=0.0)


@pytest.mark.parametrize("bc", ["zero", "reflective"])
@pytest.mark.parametrize("dtype,m,n,h", [
    ("float64", 96, 128, 6),     # DMMA persistent passes
    ("float64", 250, 202, 20),   # odd tiles, wide band
    ("float32", 96, 128, 6),     # 3xTF32 mma.sync passes
    ("float32", 4096, 4096, 16), # default policy: tcgen05 passes (2048 chunks)
])
def test_projection_mask_and_values_bit_exact(bc, dtype, m, n, h):
    rng = np.random.default_rng(m * 7 + n + (bc == "zero"))
    op = sparse_int_operator(rng, m, n, 2, bc, h)
    B = rng.integers(-3, 4, size=(m, n)).astype(np.float64)
    X0 = rng.integers(-3, 4, size=(m, n)).astype(np.float64)
    L, lam = 0.75, 0.5
    _, beta = kb.momentum_table(2)
    assert beta[0] == 0.0
    oop = C.OracleOp(op, rel_tol=0.0)
    for iters in ((1, 2) if dtype == "float64" else (1,)):
        want = C.sfista(oop, B, L, lam, iters, beta, X0=X0, project=True)
        run = kb.sfista(op, B, kb.SolveConfig(lam=lam, lipschitz=L, max_iter=iters, record_history=False),
                        X0=X0, options=kb.SolveOptions(dtype=dtype, project=True, use_graph=False))
        got = run.x
        clamped = want == 0
        assert 0.05 < clamped.mean() < 0.95  # the mask is non-trivial
        np.testing.assert_array_equal(got == 0, clamped, err_msg=f"mask, iteration {iters}")
        np.testing.assert_array_equal(got, want, err_msg=f"values, iteration {iters}")
        assert not np.any(np.signbit(got))  # -0.0 maps to +0.0 (np.maximum semantics)
    engines = device_operator(op, dtype).last_engines()
    assert "generic" not in engines or m % 2 or n % 2, engines
    if dtype == "float32" and m == 4096:
        assert engines == ["tcgen05_tf32"] * 4, engines
