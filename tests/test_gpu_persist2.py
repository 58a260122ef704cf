"""The second whole-solve persistent kernel (csrc/kb_persist2.cuh: zero BC, half widths <= 15,
r <= 4, n a multiple of 64 up to 512; cfg1's shape) against the C oracle, on both row blockings
(KB_PERSIST_RB=1: one image row per CTA, =2: two) and against the first form (KB_PERSIST2=0).

It is the default engine for these shapes, so every case also runs through the reference-facing
`sfista`; the narrow-band cases exercise the zero-padded 31-tap windows, the small-m cases the
CTAs whose staged rows are partly outside the image, and m % RB != 0 a half-empty last CTA.
"""

import os

import numpy as np
import pytest

from conftest import cuda_ok

pytestmark = pytest.mark.gpu

if not cuda_ok():  # pragma: no cover - collected on CPU but skipped
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1901_00913_b200 as kb  # noqa: E402
from oracle import kb_oracle as C  # noqa: E402
from paper_1901_00913_b200.device import device_operator  # noqa: E402


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def operator(rng, m, n, r, ha, hb, integer=False):
    ja, jb = m // 2 + 1, n // 2 + 1
    terms = []
    for _ in range(r):
        a, b = np.zeros(m), np.zeros(n)
        for c, j, h in ((a, ja, ha), (b, jb, hb)):
            lo, hi = max(0, j - 1 - h), min(len(c), j + h)
            if integer:
                c[lo:hi] = rng.integers(-2, 3, size=hi - lo)
                c[j - 1] = 1.0
            else:
                c[lo:hi] = rng.standard_normal(hi - lo) / (hi - lo)
        terms.append(kb.KronTerm(sigma=1.0, H=kb.toep(a, ja), K=kb.toep(b, jb)))
    return kb.KronOperator(terms=tuple(terms), shape=(m, n), bc=kb.BoundaryCondition.ZERO,
                           sigma=np.ones(r), s=r, rank=r, eps=0.0)


class env:
    def __init__(self, **kv):
        self.kv = kv

    def __enter__(self):
        self.old = {k: os.environ.get(k) for k in self.kv}
        os.environ.update({k: str(v) for k, v in self.kv.items()})

    def __exit__(self, *exc):
        for k, v in self.old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


CASES = [
    # m, n, r, ha, hb, iters
    (256, 256, 3, 15, 15, 40),   # cfg1's shape and band
    (256, 256, 4, 15, 7, 25),
    (200, 512, 2, 4, 15, 20),    # widest row, narrow axis-0 band
    (37, 64, 1, 15, 15, 30),     # m < 2 x 15 + RB: every CTA's window is clipped
    (129, 192, 3, 9, 12, 20),    # m odd: the last CTA owns one row at RB = 2
]


@pytest.mark.parametrize("rb", [1, 2])
@pytest.mark.parametrize("m,n,r,ha,hb,iters", CASES)
def test_persist2_matches_oracle(m, n, r, ha, hb, iters, rb):
    rng = np.random.default_rng(m * 31 + n + r)
    op = operator(rng, m, n, r, ha, hb)
    B = rng.random((m, n))
    oop = C.OracleOp(op)
    L = 1.05 * float(np.sum([np.abs(t.H.c).sum() * np.abs(t.K.c).sum() for t in op.terms])) ** 2 / r
    lam = 0.05
    _, beta = kb.momentum_table(iters)
    for project in (True, False):
        want = C.sfista(oop, B, L, lam, iters, beta, project=project)
        cfg = kb.SolveConfig(lam=lam, lipschitz=L, max_iter=iters, record_history=False)
        with env(KB_PERSIST_RB=rb):
            got = kb.sfista(op, B, cfg, options=kb.SolveOptions(dtype="float64", project=project, use_graph=False)).x
        assert device_operator(op, "float64").last_engines() == ["persist_f64"] * 4
        assert rel(got, want) <= 1e-10, (project, rel(got, want))
        with env(KB_PERSIST2=0, KB_PERSIST_RB=rb):
            first = kb.sfista(op, B, cfg, options=kb.SolveOptions(dtype="float64", project=project,
                                                                   use_graph=False)).x
        assert rel(got, first) <= 1e-11


def test_persist2_two_ctas_per_sm():
    """512 x 256: 256 CTAs at two rows each, two per SM -- the instantiation without
    register-resident B fragments (the ~200-register one fits one CTA per SM only)."""
    m, n, r, iters = 512, 256, 3, 12
    rng = np.random.default_rng(5)
    op = operator(rng, m, n, r, 15, 15)
    B = rng.random((m, n))
    L = 1.05 * float(np.sum([np.abs(t.H.c).sum() * np.abs(t.K.c).sum() for t in op.terms])) ** 2 / r
    _, beta = kb.momentum_table(iters)
    want = C.sfista(C.OracleOp(op), B, L, 0.05, iters, beta, project=True)
    cfg = kb.SolveConfig(lam=0.05, lipschitz=L, max_iter=iters, record_history=False)
    got = kb.sfista(op, B, cfg, options=kb.SolveOptions(dtype="float64", project=True, use_graph=False)).x
    assert device_operator(op, "float64").last_engines() == ["persist_f64"] * 4
    assert rel(got, want) <= 1e-10
    with env(KB_PERSIST2=0):
        first = kb.sfista(op, B, cfg, options=kb.SolveOptions(dtype="float64", project=True, use_graph=False)).x
    assert rel(got, first) <= 1e-11


@pytest.mark.parametrize("sync", ["flags", "counter"])
@pytest.mark.parametrize("m,n,r,ha,hb,iters", [CASES[0], CASES[3], CASES[4]])
def test_persist2_other_synchronisations_match_grid_barrier(m, n, r, ha, hb, iters, sync):
    """KB_PERSIST2_SYNC=flags (neighbour phase epochs, one 128-byte line per CTA) and =counter (one
    release/acquire arrival counter) order the same memory operations as the cooperative grid
    barrier: the solves must agree bit for bit (same arithmetic, only the waiting differs), over
    enough iterations for a missed wait to show, twice (the flags are re-zeroed per launch)."""
    rng = np.random.default_rng(11 * m + n)
    op = operator(rng, m, n, r, ha, hb)
    B = rng.random((m, n))
    L = 1.05 * float(np.sum([np.abs(t.H.c).sum() * np.abs(t.K.c).sum() for t in op.terms])) ** 2 / r
    cfg = kb.SolveConfig(lam=0.05, lipschitz=L, max_iter=3 * iters, record_history=False)
    opts = kb.SolveOptions(dtype="float64", project=True, use_graph=False)
    with env(KB_PERSIST2_SYNC="grid"):
        want = kb.sfista(op, B, cfg, options=opts).x
    for _ in range(2):
        with env(KB_PERSIST2_SYNC=sync):
            got = kb.sfista(op, B, cfg, options=opts).x
        np.testing.assert_array_equal(got, want)
    assert device_operator(op, "float64").last_engines() == ["persist_f64"] * 4


@pytest.mark.parametrize("rb", [1, 2])
def test_persist2_bit_exact_on_integers(rb):
    """Integer generators and data with L + lam^2 = 1: the first two iterations are exact (see
    test_gpu_projection.py), so the DMMA axis-1 sums and the register-resident x / y must equal
    the C oracle bit for bit, clamp mask included."""
    rng = np.random.default_rng(7 + rb)
    m = n = 256
    op = operator(rng, m, n, 3, 15, 15, integer=True)
    B = rng.integers(-3, 4, size=(m, n)).astype(np.float64)
    X0 = rng.integers(-3, 4, size=(m, n)).astype(np.float64)
    L, lam = 0.75, 0.5
    _, beta = kb.momentum_table(2)
    oop = C.OracleOp(op, rel_tol=0.0)
    for iters in (1, 2):
        want = C.sfista(oop, B, L, lam, iters, beta, X0=X0, project=True)
        with env(KB_PERSIST_RB=rb):
            got = kb.sfista(op, B, kb.SolveConfig(lam=lam, lipschitz=L, max_iter=iters, record_history=False),
                            X0=X0, options=kb.SolveOptions(dtype="float64", project=True, use_graph=False)).x
        assert 0.05 < (want == 0).mean() < 0.95
        np.testing.assert_array_equal(got, want)
        assert not np.any(np.signbit(got))
    assert device_operator(op, "float64").last_engines() == ["persist_f64"] * 4


def test_persist2_nonfinite_detected():
    """A NaN in B reaches every x through the solve; the kernel's per-iteration non-finite flag
    must report it the same way as the first form (NumericError from sfista)."""
    rng = np.random.default_rng(3)
    m = n = 128
    op = operator(rng, m, n, 2, 10, 10)
    B = rng.random((m, n))
    B[60, 60] = np.nan
    cfg = kb.SolveConfig(lam=0.05, lipschitz=2.0, max_iter=5, record_history=False)
    errs = []
    for flag in ("1", "0"):
        with env(KB_PERSIST2=flag):
            try:
                kb.sfista(op, B, cfg, options=kb.SolveOptions(dtype="float64", project=False, use_graph=False))
                errs.append(None)
            except Exception as e:  # noqa: BLE001 - the same class and message either way
                errs.append((type(e).__name__, str(e)))
    assert errs[0] == errs[1] and errs[0] is not None
