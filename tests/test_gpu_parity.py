"""GPU parity of the B200 path against the CPU oracle (oracle/kronblur_port.py).

Tolerances (north_star): fp64 relative Frobenius <= 1e-10 (operator applications: 1e-12),
fp32 <= 1e-4 plus PSNR within 0.01 dB; boundary / projection index logic bit-exact on
integer-valued inputs (exact through the dense index rules).
"""

import numpy as np
import pytest

from conftest import blur_loop, cuda_ok, hankel_loop, random_psf, toeplitz_loop

pytestmark = pytest.mark.gpu

if not cuda_ok():  # pragma: no cover - collected on CPU but skipped
    pytest.skip("needs a CUDA device", allow_module_level=True)

import torch  # noqa: E402

import paper_1901_00913_b200 as kb  # noqa: E402
from oracle import kronblur_port as port  # noqa: E402

ZERO = kb.BoundaryCondition.ZERO
REFL = kb.BoundaryCondition.REFLECTIVE


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(np.asarray(b)), 1e-300))


def int_operator(rng, m, n, r, bc, ha, hb, lo=-5, hi=5):
    """KronOperator with integer generators: exact arithmetic in fp64 for |values| small."""
    make = kb.toep if bc == "zero" else kb.toep_plus_hank
    terms = []
    ja, jb = int(rng.integers(1, m + 1)), int(rng.integers(1, n + 1))
    for _ in range(r):
        a = np.zeros(m)
        b = np.zeros(n)
        for d in range(-ha, ha + 1):
            if 1 <= ja + d <= m:
                a[ja + d - 1] = rng.integers(lo, hi + 1)
        for d in range(-hb, hb + 1):
            if 1 <= jb + d <= n:
                b[jb + d - 1] = rng.integers(lo, hi + 1)
        terms.append(kb.KronTerm(sigma=1.0, H=make(a, ja), K=make(b, jb)))
    return kb.KronOperator(terms=tuple(terms), shape=(m, n), bc=kb.BoundaryCondition(bc),
                           sigma=np.ones(r), s=r, rank=r, eps=0.0)


# ----------------------------------------------------------------- index logic, bit exact
@pytest.mark.parametrize("bc", ["zero", "reflective"])
@pytest.mark.parametrize("shape,r,ha,hb", [((7, 9), 2, 3, 2), ((33, 40), 3, 6, 6),
                                            ((70, 65), 4, 12, 9), ((129, 300), 5, 31, 20),
                                            ((5, 5), 1, 4, 4), ((1, 17), 2, 0, 5)])
def test_integer_apply_bit_exact(bc, shape, r, ha, hb, rng):
    m, n = shape
    op = int_operator(rng, m, n, r, bc, min(ha, m - 1), min(hb, n - 1))
    X = rng.integers(-7, 8, size=(m, n)).astype(float)
    want = port.dense_kron_apply(op, X)
    wantT = port.dense_kron_apply(op, X, adjoint=True)
    assert np.array_equal(kb.kron_apply(op, X), want)
    assert np.array_equal(kb.kron_apply_adjoint(op, X), wantT)


def test_dense_factors_match_loop_oracles(rng):
    for _ in range(20):
        n = int(rng.integers(1, 30))
        j = int(rng.integers(1, n + 1))
        c = rng.integers(-9, 10, size=n).astype(float)
        assert np.array_equal(port.dense_toeplitz(c, j), toeplitz_loop(c, j))
        assert np.array_equal(port.dense_hankel(c, j), hankel_loop(c, j))


@pytest.mark.parametrize("bc", ["zero", "reflective"])
def test_untruncated_apply_equals_direct_blur(bc, rng):
    # kron_apply on the full expansion is the exact blur (test_kron.py:142-152)
    for size in (3, 5, 7):
        psf = random_psf(rng, size)
        m = 12
        op = kb.decompose(psf, kb.BoundaryCondition(bc), shape=(m, m))
        padded = kb.pad_to(psf, m, m)
        X = rng.standard_normal((m, m))
        want = blur_loop(padded.values, padded.center, X, bc)
        got = kb.kron_apply(op, X)
        assert np.max(np.abs(got - want)) <= 1e-10 * max(1.0, np.max(np.abs(want)))


# ----------------------------------------------------------------- fp64 operator parity
@pytest.mark.parametrize("bc", [ZERO, REFL])
@pytest.mark.parametrize("m,size,s", [(64, 9, 3), (256, 31, 3), (200, 15, 4), (96, 63, 5)])
def test_apply_matches_oracle_fp64(bc, m, size, s, rng):
    psf = random_psf(rng, size)
    op = kb.decompose(psf, bc, s=s, shape=(m, m))
    pop = port.PortOperator(op)
    X = rng.standard_normal((m, m))
    assert rel(kb.kron_apply(op, X), port.kron_apply(pop, X)) <= 1e-12
    assert rel(kb.kron_apply_adjoint(op, X), port.kron_apply_adjoint(pop, X)) <= 1e-12


@pytest.mark.parametrize("exact", [False, True])
@pytest.mark.parametrize("name", ["cfg1", "cfg2", "cfg5"])
def test_symmetric_generators_sign_fill(name, exact, monkeypatch):
    # centrally symmetric BASELINE PSFs give (anti)symmetric generators: the adjoint folds via
    # sign-reflected tile fills; KB_EXACT_FOLD=1 forces the exact fold kernels instead
    from paper_1901_00913_b200 import workloads as W
    from paper_1901_00913_b200.device import DeviceOperator

    cfg = W.CONFIGS[name]
    m = 3 * cfg.w + 7
    bc = kb.BoundaryCondition("reflective")  # exercise the fold on every PSF family
    op = kb.decompose(W.make_psf(cfg), bc, s=cfg.r, shape=(m, m))
    if exact:
        monkeypatch.setenv("KB_EXACT_FOLD", "1")
    info = DeviceOperator([op], "float64").info()
    assert info["sym_a"] == info["sym_b"] == (0 if exact else 1)
    dev = DeviceOperator([op], "float64")
    rng = np.random.default_rng(3)
    X = rng.standard_normal((m, m))
    t = torch.from_numpy(X).cuda()
    pop = port.PortOperator(op)
    assert rel(dev.apply(t, adjoint=True).cpu().numpy(), port.kron_apply_adjoint(pop, X)) <= 1e-12
    assert rel(dev.apply(t).cpu().numpy(), port.kron_apply(pop, X)) <= 1e-12


@pytest.mark.parametrize("bc", [ZERO, REFL])
def test_adjoint_identity(bc, rng):
    psf = random_psf(rng, 11)
    op = kb.decompose(psf, bc, s=4, shape=(150, 150))
    X = rng.standard_normal((150, 150))
    Y = rng.standard_normal((150, 150))
    lhs = float(np.vdot(kb.kron_apply(op, X), Y))
    rhs = float(np.vdot(X, kb.kron_apply_adjoint(op, Y)))
    assert abs(lhs - rhs) <= 1e-11 * max(1.0, abs(lhs))


def test_apply_is_linear(rng):
    psf = random_psf(rng, 7)
    op = kb.decompose(psf, REFL, s=3, shape=(80, 80))
    X, Y = rng.standard_normal((2, 80, 80))
    lhs = kb.kron_apply(op, 2.5 * X - 1.25 * Y)
    rhs = 2.5 * kb.kron_apply(op, X) - 1.25 * kb.kron_apply(op, Y)
    assert np.max(np.abs(lhs - rhs)) <= 1e-12 * max(1.0, np.max(np.abs(lhs)))


def test_fp32_apply(rng):
    psf = random_psf(rng, 31)
    op = kb.decompose(psf, REFL, s=5, shape=(300, 300))
    X = rng.standard_normal((300, 300))
    got = kb.kron_apply(op, X, dtype="float32")
    assert rel(got, port.kron_apply(port.PortOperator(op), X)) <= 1e-5


def test_tensor_in_tensor_out(rng):
    psf = random_psf(rng, 5)
    op = kb.decompose(psf, ZERO, s=2, shape=(40, 40))
    X = rng.standard_normal((40, 40))
    t = torch.from_numpy(X).cuda()
    out = kb.kron_apply(op, t)
    assert isinstance(out, torch.Tensor) and out.is_cuda
    assert rel(out.cpu().numpy(), port.kron_apply(port.PortOperator(op), X)) <= 1e-12


def test_shape_mismatch_raises(rng):
    op = kb.decompose(random_psf(rng, 3), ZERO, s=1, shape=(8, 8))
    with pytest.raises(kb.ArgumentError):
        kb.kron_apply(op, np.zeros((8, 9)))


# ----------------------------------------------------------------- solver parity
@pytest.mark.parametrize("bc", [ZERO, REFL])
@pytest.mark.parametrize("project", [False, True])
def test_sfista_matches_oracle_fp64(bc, project, rng):
    psf = random_psf(rng, 15)
    m = 128
    op = kb.decompose(psf, bc, s=3, shape=(m, m))
    B = rng.random((m, m)) - 0.2
    L = port.estimate_lipschitz(lambda v: port.kron_apply(port.PortOperator(op), v),
                                lambda v: port.kron_apply_adjoint(port.PortOperator(op), v), (m, m), 30, 3)
    cfg = kb.SolveConfig(lam=0.05, lipschitz=L, max_iter=40, record_history=False)
    run = kb.sfista(op, B, cfg, options=kb.SolveOptions(project=project))
    want, _ = port.sfista(op, B, L, 0.05, 40, project=project)
    assert run.iterations == 40
    assert rel(run.x, want) <= 1e-10
    if project:
        assert np.all(run.x >= 0)


def test_sfista_iterates_and_history_match_oracle(rng):
    psf = random_psf(rng, 5)
    op = kb.decompose(psf, REFL, s=3, shape=(16, 16))
    B = rng.standard_normal((16, 16))
    cfg = kb.SolveConfig(lam=0.15, lipschitz=2.0, max_iter=35, record_iterates=True)
    run = kb.sfista(op, B, cfg)
    _, its = port.sfista(op, B, 2.0, 0.15, 35, record_iterates=True)
    assert len(run.iterates) == 35 and len(run.history) == 35
    for a, b in zip(run.iterates, its):
        assert np.max(np.abs(a - b)) <= 1e-12 * max(1.0, np.max(np.abs(b)))
    assert [h.k for h in run.history] == list(range(1, 36))
    assert abs(run.history[1].t - 1.61803398874989484820458) < 1e-14
    pop = port.PortOperator(op)
    r = port.kron_apply(pop, its[-1]) - B
    phi = 0.5 * float(r.ravel() @ r.ravel()) + 0.5 * 0.15**2 * float(its[-1].ravel() @ its[-1].ravel())
    assert abs(run.history[-1].objective - phi) <= 1e-12 * abs(phi)


def test_sfista_identity_operator_gives_half_b(rng):
    from paper_1901_00913_b200 import Psf

    op = kb.decompose(Psf(np.ones((1, 1)), (1, 1)), ZERO, shape=(6, 6))
    B = rng.standard_normal((6, 6))
    run = kb.sfista(op, B, kb.SolveConfig(lam=1.0, lipschitz=1.05, max_iter=200))
    assert np.max(np.abs(run.x - B / 2.0)) < 1e-9


def test_divergence_raises_numeric_error(rng):
    op = kb.decompose(random_psf(rng, 3), ZERO, s=1, shape=(8, 8))
    B = rng.standard_normal((8, 8)) * 100
    cfg = kb.SolveConfig(lam=1e-3, lipschitz=1e-6, max_iter=400, record_history=False)
    with pytest.raises(kb.NumericError, match="non-finite iterate at iteration"):
        kb.sfista(op, B, cfg)


def test_projection_keeps_nan_visible():
    # F3: the clamp must propagate NaN so the non-finite check still fires
    op = kb.decompose(kb.Psf(np.ones((1, 1)), (1, 1)), ZERO, shape=(4, 4))
    B = np.zeros((4, 4))
    B[1, 2] = np.nan
    cfg = kb.SolveConfig(lam=1.0, lipschitz=1.05, max_iter=3, record_history=False)
    with pytest.raises(kb.NumericError, match="iteration 1"):
        kb.sfista(op, B, cfg, options=kb.SolveOptions(project=True))


def test_x0_shape_mismatch(rng):
    op = kb.decompose(random_psf(rng, 3), ZERO, s=1, shape=(8, 8))
    with pytest.raises(kb.ArgumentError):
        kb.sfista(op, np.zeros((8, 8)), kb.SolveConfig(lam=0.1, lipschitz=1.0), X0=np.zeros((7, 8)))


def test_graph_and_plain_paths_agree(rng):
    psf = random_psf(rng, 9)
    op = kb.decompose(psf, REFL, s=3, shape=(96, 96))
    B = rng.random((96, 96))
    cfg = kb.SolveConfig(lam=0.05, lipschitz=1.2, max_iter=25, record_history=False)
    a = kb.sfista(op, B, cfg, options=kb.SolveOptions(use_graph=True)).x
    b = kb.sfista(op, B, cfg, options=kb.SolveOptions(use_graph=False)).x
    assert np.array_equal(a, b)


# ----------------------------------------------------------------- Lipschitz
@pytest.mark.parametrize("bc", [ZERO, REFL])
@pytest.mark.parametrize("form", ["matrix", "vector"])
def test_power_iteration_matches_oracle(bc, form, rng):
    psf = random_psf(rng, 7)
    m = 48
    op = kb.decompose(psf, bc, s=3, shape=(m, m))
    pop = port.PortOperator(op)
    if form == "matrix":
        want = port.estimate_lipschitz(lambda v: port.kron_apply(pop, v),
                                       lambda v: port.kron_apply_adjoint(pop, v), (m, m), 50, 4)
    else:
        want = port.estimate_lipschitz(
            lambda v: kb.vec(port.kron_apply(pop, kb.unvec(v, m, m))),
            lambda v: kb.vec(port.kron_apply_adjoint(pop, kb.unvec(v, m, m))), m * m, 50, 4)
    apply, adjoint = kb.make_ops(op, form=form)
    got = kb.estimate_lipschitz(apply, adjoint, (m, m) if form == "matrix" else m * m, iters=50, seed=4)
    assert abs(got - want) <= 1e-12 * want


def test_power_iteration_zero_operator_warns():
    op = int_operator(np.random.default_rng(0), 6, 6, 1, "zero", 1, 1, 0, 0)
    with pytest.warns(UserWarning, match="zero"):
        L = kb.lipschitz(op, iters=5)
    assert 0 < L < 1e-10


# ----------------------------------------------------------------- batch (cfg3 shape class)
def test_batched_solve_matches_per_image(rng):
    from paper_1901_00913_b200.device import DeviceOperator

    ops, Bs, Ls = [], [], []
    for i in range(3):
        psf = random_psf(rng, 7)
        op = kb.decompose(psf, ZERO, s=2, shape=(40, 40))
        ops.append(op)
        Bs.append(rng.random((40, 40)))
        Ls.append(1.0 + 0.1 * i)
    dev = DeviceOperator(ops, "float64")
    x, _ = kb.sfista_batch(dev, np.stack(Bs), np.array(Ls), 0.02, 30,
                           options=kb.SolveOptions(project=True))
    for i in range(3):
        want, _ = port.sfista(ops[i], Bs[i], Ls[i], 0.02, 30, project=True)
        assert rel(x[i], want) <= 1e-10


@pytest.mark.parametrize("dtype", ["float64", "float32"])
@pytest.mark.parametrize("orient", [0, 1])
def test_mixed_axis_symmetry(dtype, orient, rng):
    # one axis (anti)symmetric, the other general: the split pass stores Z^T's reflected halo
    # rows while the other axis takes the exact fold kernels (which must keep the halo in step)
    from paper_1901_00913_b200 import Psf
    from paper_1901_00913_b200.device import DeviceOperator

    u = np.array([1.0, 3.0, 5.0, 3.0, 1.0])
    v = rng.random(5) + 0.1
    vals = np.outer(u, v) if orient == 0 else np.outer(v, u)
    op = kb.decompose(Psf(vals / vals.sum(), (3, 3)), REFL, s=1, shape=(64, 64))
    info = DeviceOperator([op], dtype).info()
    assert info["sym_a"] != info["sym_b"]
    X = rng.standard_normal((64, 64))
    pop = port.PortOperator(op)
    tol = 1e-12 if dtype == "float64" else 1e-5
    assert rel(kb.kron_apply_adjoint(op, X, dtype=dtype), port.kron_apply_adjoint(pop, X)) <= tol
    assert rel(kb.kron_apply(op, X, dtype=dtype), port.kron_apply(pop, X)) <= tol


@pytest.mark.parametrize("dtype", ["float64", "float32"])
def test_misaligned_device_buffers(dtype):
    # views 8 bytes off a 16-byte boundary cannot feed TMA / vector epilogues: the generic
    # kernels take over (and the sum pass must not expect reflected halo rows)
    from paper_1901_00913_b200.device import DeviceOperator

    rng = np.random.default_rng(11)
    m = 96
    op = kb.decompose(random_psf(rng, 9), REFL, s=3, shape=(m, m))
    X = rng.standard_normal((m, m))
    td = torch.float64 if dtype == "float64" else torch.float32
    dev = DeviceOperator([op], dtype)
    base = torch.zeros(m * m + 4, dtype=td, device="cuda")
    off = 1 if dtype == "float64" else 2
    xv = base[off:off + m * m].view(m, m)
    xv.copy_(torch.from_numpy(X))
    pop = port.PortOperator(op)
    tol = 1e-12 if dtype == "float64" else 1e-5
    xa = torch.from_numpy(X).to("cuda", td)
    obase = torch.zeros(m * m + 4, dtype=td, device="cuda")
    ov = obase[off:off + m * m].view(m, m)
    for adjoint in (False, True):
        want = port.kron_apply_adjoint(pop, X) if adjoint else port.kron_apply(pop, X)
        got = dev.apply(xv, adjoint=adjoint).double().cpu().numpy()  # misaligned operand
        assert rel(got, want) <= tol
        dev.apply(xa, out=ov, adjoint=adjoint)  # aligned operand, misaligned result
        assert rel(ov.double().cpu().numpy(), want) <= tol


# ----------------------------------------------------------------- full-rank operators
@pytest.mark.parametrize("bc", [ZERO, REFL])
@pytest.mark.parametrize("dtype", ["float64", "float32"])
def test_full_rank_operator_matches_oracle(rng, bc, dtype):
    """restore(s=None) decomposes the padded PSF at full rank (pipeline.py:169, rank up to the PSF
    size): 41 terms here, beyond the BASELINE r <= 10 configs."""
    psf = random_psf(rng, 41)
    op = kb.decompose(psf, bc, shape=(96, 96))
    assert len(op.terms) == 41
    pop = port.PortOperator(op)
    X = rng.standard_normal((96, 96))
    tol = 1e-12 if dtype == "float64" else 1e-5
    if dtype == "float64":
        assert rel(kb.kron_apply(op, X), port.kron_apply(pop, X)) <= tol
        assert rel(kb.kron_apply_adjoint(op, X), port.kron_apply_adjoint(pop, X)) <= tol
    B = port.kron_apply(pop, np.abs(X))
    cfg = kb.SolveConfig(lam=0.05, lipschitz=1.05, max_iter=20, record_history=False)
    run = kb.sfista(op, B, cfg, options=kb.SolveOptions(dtype=dtype))
    want, _ = port.sfista(op, B, 1.05, 0.05, 20)
    assert rel(run.x, want) <= (1e-10 if dtype == "float64" else 1e-4)


def test_sfista_accepts_cuda_tensors(rng):
    """Optional extension: device tensors in skip the host copies; same result."""
    psf = random_psf(rng, 7)
    op = kb.decompose(psf, REFL, s=3, shape=(64, 64))
    B = rng.random((64, 64))
    X0 = 0.1 * rng.random((64, 64))
    cfg = kb.SolveConfig(lam=0.05, lipschitz=1.2, max_iter=20, record_history=False)
    host = kb.sfista(op, B, cfg, X0=X0).x
    dev = kb.sfista(op, torch.from_numpy(B).cuda(), cfg, X0=torch.from_numpy(X0).cuda()).x
    assert isinstance(dev, torch.Tensor) and dev.is_cuda and dev.dtype == torch.float64
    assert np.array_equal(dev.cpu().numpy(), host)
    hist = kb.sfista(op, torch.from_numpy(B).cuda(), kb.SolveConfig(lam=0.05, lipschitz=1.2, max_iter=5))
    assert isinstance(hist.x, np.ndarray) and len(hist.history) == 5
