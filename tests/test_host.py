"""Host-side logic of the drop-in (no GPU): C-ABI exports, band extraction, setup, validation."""

import ctypes
import os
import re
import warnings

import numpy as np
import pytest

from conftest import ROOT, cuda_ok, random_psf

import paper_1901_00913_b200 as kb
from paper_1901_00913_b200 import device, structured, workloads
from oracle import kronblur_port as port

HEADER = os.path.join(ROOT, "include", "kronblur_b200.h")


def header_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(kb_[a-z_0-9]+)\s*\(", text)))


def test_library_exports_every_header_symbol():
    if not os.path.exists(device.LIB_PATH):
        pytest.skip("extension not built (run __graft_entry__.build())")
    lib = ctypes.CDLL(device.LIB_PATH)
    names = header_functions()
    assert len(names) >= 12
    for name in names:
        assert hasattr(lib, name), name
    # the Python binding declares exactly the header's functions
    assert sorted(device.EXPORTS) == names
    lib2 = device.load_library()
    assert lib2.kb_version().decode().startswith("kronblur_b200")
    assert lib2.kb_max_half_width() >= 512
    assert lib2.kb_last_error() == b""


def test_no_cpu_fallback_without_cuda():
    if cuda_ok():
        pytest.skip("a GPU is present")
    op = kb.decompose(kb.Psf(np.ones((1, 1)), (1, 1)), kb.BoundaryCondition.ZERO, shape=(4, 4))
    with pytest.raises(RuntimeError, match="CUDA"):
        kb.kron_apply(op, np.zeros((4, 4)))
    with pytest.raises(RuntimeError, match="CUDA"):
        kb.sfista(op, np.zeros((4, 4)), kb.SolveConfig(lam=1.0, lipschitz=1.0, max_iter=2))


def test_factor_band_is_the_stencil():
    c = np.array([0, 0, 3.0, -1.0, 2.0, 0, 0, 5.0, 0])
    f = kb.toep(c, 4)  # anchor j=4 -> c_d = c[4+d]
    dlo, taps = kb.factor_band(f)
    assert dlo == -1 and taps.tolist() == [3.0, -1.0, 2.0, 0, 0, 5.0]
    # stencil form reproduces the dense matrix: y[s] = sum_d c_d x[s-d]
    n = c.size
    D = kb.factor_to_dense(f)
    x = np.arange(1.0, n + 1)
    y = np.zeros(n)
    for s in range(n):
        for t, cd in enumerate(taps):
            d = dlo + t
            if 0 <= s - d < n:
                y[s] += cd * x[s - d]
    assert np.array_equal(D @ x, y)
    # leakage below the tolerance is trimmed, exact zeros always
    c2 = c.copy()
    c2[0] = 1e-17
    assert kb.factor_band(kb.toep(c2, 4), 1e-14)[0] == -1
    assert kb.factor_band(kb.toep(c2, 4), 0.0)[0] == -3


def test_structured_validation():
    with pytest.raises(kb.ArgumentError):
        kb.toep([1.0, 2.0], 0)
    with pytest.raises(kb.ArgumentError):
        kb.toep([1.0, 2.0], 3)
    with pytest.raises(kb.ArgumentError):
        kb.hank([], 1)
    with pytest.raises(kb.ArgumentError):
        kb.toep([1.0, np.nan], 1)
    f = kb.toep([1.0, 2.0, 3.0], 2)
    with pytest.raises(ValueError):
        f.c[0] = 9.0
    with pytest.raises(kb.CapacityError):
        kb.factor_to_dense(kb.toep(np.ones(5000), 1))


def test_axis_band_unification_and_kinds():
    rng = np.random.default_rng(0)
    fs = [kb.toep(np.r_[np.zeros(3), rng.standard_normal(3), np.zeros(4)], 5),
          kb.toep(np.r_[np.zeros(1), rng.standard_normal(5), np.zeros(4)], 5)]
    dlo, taps, bc = device._axis_bands(fs, 0.0)
    assert bc == device.KB_BC_ZERO and dlo == -3 and taps.shape == (2, 5)
    with pytest.raises(kb.ArgumentError):
        device._axis_bands([kb.hank(np.ones(4), 2)], 0.0)
    with pytest.raises(kb.ArgumentError):
        device._axis_bands([kb.toep(np.ones(4), 2), kb.toep_plus_hank(np.ones(4), 2)], 0.0)


def test_momentum_table_matches_engine_recurrence():
    ts, beta = kb.momentum_table(50)
    t = 1.0
    for k in range(50):
        tn = port.momentum_next(t)
        assert ts[k] == t and beta[k] == (t - 1.0) / tn
        t = tn
    with pytest.raises(kb.ArgumentError):
        kb.momentum_next(0.9)


def test_lipschitz_start_vectors_match_reference_streams():
    from paper_1901_00913_b200.solvers import _start_vector

    v = _start_vector(7, 5, 6, "matrix")
    assert np.array_equal(v, port.lipschitz_start(7, (5, 6)))
    w = _start_vector(7, 5, 6, "vector")
    assert np.array_equal(w, kb.unvec(port.lipschitz_start(7, 30), 5, 6))


def test_generic_estimate_lipschitz_known_answers():
    # solvers.py host loop for non-GPU callables (test_solvers.py:69-79 known answers)
    L = kb.estimate_lipschitz(lambda x: x, lambda y: y, 8)
    assert L == pytest.approx(kb.LIPSCHITZ_SAFETY, rel=1e-12)
    A = np.diag([2.0, 1.0])
    L = kb.estimate_lipschitz(lambda x: A @ x, lambda y: A.T @ y, 2)
    assert L == pytest.approx(4.0 * kb.LIPSCHITZ_SAFETY, rel=1e-9)
    with warnings.catch_warnings(record=True) as caught:
        warnings.simplefilter("always")
        L = kb.estimate_lipschitz(lambda x: 0 * x, lambda y: 0 * y, 4)
    assert 0 < L < 1e-10 and any("zero" in str(w.message) for w in caught)


def test_power_history_rules():
    from paper_1901_00913_b200.solvers import _finish_power

    h = np.array([[2.0, 4.0], [3.0, 9.0]])
    assert _finish_power(h) == pytest.approx(3.0 * 1.05)
    with pytest.warns(UserWarning):
        assert _finish_power(np.array([[1.0, 1.0], [0.0, 0.0]])) < 1e-10


def test_solveconfig_validation():
    with pytest.raises(kb.ArgumentError):
        kb.SolveConfig(lam=-1.0, lipschitz=1.0)
    with pytest.raises(kb.ArgumentError):
        kb.SolveConfig(lam=0.1, lipschitz=0.0)
    with pytest.raises(kb.ArgumentError):
        kb.SolveConfig(lam=0.1, lipschitz=1.0, max_iter=0)
    with pytest.raises(kb.ArgumentError):
        kb.SolveConfig(lam=0.1, lipschitz=1.0, rel_tol=-1)


def test_decompose_edge_cases(rng):
    p = kb.psf_gaussian(5, 1.2) if hasattr(kb, "psf_gaussian") else None
    vals = np.outer(np.hanning(7)[1:-1], np.hanning(7)[1:-1])
    psf = kb.Psf(vals / vals.sum(), (3, 3))
    op = kb.decompose(psf, kb.BoundaryCondition.ZERO, shape=(9, 9))
    assert op.rank == 1 and op.s == 1  # separable
    op4 = kb.decompose(psf, kb.BoundaryCondition.ZERO, s=4, shape=(9, 9))  # beyond the block: full SVD
    assert len(op4.terms) == 4 and op4.sigma[1] <= 1e-12 * op4.sigma[0]
    assert op4.truncate(2).s == 2 and op4.truncate(2).eps >= op4.eps - 1e-15
    with pytest.raises(kb.ArgumentError):
        op4.truncate(5)
    with pytest.raises(kb.ArgumentError):
        kb.decompose(psf, kb.BoundaryCondition.ZERO, s=0, shape=(9, 9))
    with pytest.raises(kb.ArgumentError):
        kb.decompose(psf, kb.BoundaryCondition.ZERO, s=10, shape=(9, 9))
    assert p is None or p.shape == (5, 5)


@pytest.mark.parametrize("bc", ["zero", "reflective"])
def test_decompose_reconstructs_operator(bc, rng):
    psf = random_psf(rng, 5)
    op = kb.decompose(psf, kb.BoundaryCondition(bc), shape=(10, 10))
    full = port.dense_kron_apply
    X = rng.standard_normal((10, 10))
    from conftest import blur_loop

    padded = kb.pad_to(psf, 10, 10)
    want = blur_loop(padded.values, padded.center, X, bc)
    np.testing.assert_allclose(full(op, X), want, rtol=0, atol=1e-12)


def test_psf_validation_and_padding():
    with pytest.raises(kb.ArgumentError):
        kb.Psf(np.ones((2, 2)), (1, 1))  # does not sum to one
    with pytest.raises(kb.ArgumentError):
        kb.Psf(np.array([[0.5, 0.5]]), (2, 1))
    p = kb.pad_to(kb.Psf(np.full((3, 3), 1 / 9), (2, 2)), 8, 8)
    assert p.center == (5, 5) and p.values[3:6, 3:6].sum() == pytest.approx(1.0)
    with pytest.raises(kb.ArgumentError):
        kb.pad_to(kb.Psf(np.full((3, 3), 1 / 9), (2, 2)), 2, 8)
    X = np.arange(12.0).reshape(3, 4)
    assert np.array_equal(kb.unvec(kb.vec(X), 3, 4), X)


def test_workloads_are_deterministic_and_sized():
    cfg = workloads.CONFIGS["cfg1"]
    X1, psf, B1 = workloads.make_image_data(cfg, seed=3, m=64, counts=(10, 5))
    X2, _, B2 = workloads.make_image_data(cfg, seed=3, m=64, counts=(10, 5))
    assert np.array_equal(X1, X2) and np.array_equal(B1, B2)
    assert X1.shape == (64, 64) and 0 <= X1.min() and X1.max() <= 1
    assert abs(psf.values.sum() - 1) < 1e-12 and psf.values.shape == (31, 31) and psf.center == (16, 16)
    b = workloads.blur_exact(__import__("torch").from_numpy(X1), psf, cfg.bc).numpy()
    noise = np.linalg.norm(B1 - b) / np.linalg.norm(b)
    assert noise == pytest.approx(cfg.noise, rel=1e-10)
    for name in ("cfg2", "cfg3", "cfg4", "cfg5"):
        c = workloads.CONFIGS[name]
        p = workloads.make_psf(c)
        assert p.values.shape == (c.w, c.w) and abs(p.values.sum() - 1) < 1e-12


def test_blur_exact_matches_loop_oracle(rng):
    from conftest import blur_loop
    import torch

    psf = random_psf(rng, 5)
    X = rng.standard_normal((9, 11))
    for bc in ("zero", "reflective"):
        got = workloads.blur_exact(torch.from_numpy(X), psf, bc).numpy()
        np.testing.assert_allclose(got, blur_loop(psf.values, psf.center, X, bc), rtol=0, atol=1e-12)


def _stub_kronblur():
    """A stand-in package with the reference's module layout and by-name bindings (no import of
    kronblur itself), so install() is tested in every environment."""
    import sys
    import types
    from dataclasses import dataclass, field

    pkg = types.ModuleType("kbstub")
    pkg.__path__ = []
    mods = {name: types.ModuleType(f"kbstub.{name}") for name in ("solvers", "kron", "pipeline", "psf", "imaging")}

    @dataclass(frozen=True)
    class IterationRecord:
        k: int
        t: float
        objective: float
        eta: object
        gamma: object
        ms: float

    @dataclass
    class SolveRun:
        x: object
        iterations: int
        solve_ms: float
        history: list = field(default_factory=list)
        iterates: list = field(default_factory=list)

    orig = {name: (lambda *a, **k: "reference") for name in
            ("sfista", "kron_apply", "kron_apply_adjoint", "estimate_lipschitz", "decompose", "_vec_ops",
             "blur_direct", "select_lambda")}
    mods["solvers"].IterationRecord, mods["solvers"].SolveRun = IterationRecord, SolveRun
    for name in ("sfista", "kron_apply", "kron_apply_adjoint", "estimate_lipschitz", "select_lambda"):
        setattr(mods["solvers"], name, orig[name])
    for name in ("decompose", "kron_apply", "kron_apply_adjoint"):
        setattr(mods["kron"], name, orig[name])
    for name in orig:
        setattr(mods["pipeline"], name, orig[name])
    mods["psf"].blur_direct = orig["blur_direct"]
    mods["imaging"].blur_direct = orig["blur_direct"]
    for name in ("sfista", "kron_apply", "kron_apply_adjoint", "estimate_lipschitz", "decompose", "blur_direct"):
        setattr(pkg, name, orig[name])
    sys.modules["kbstub"] = pkg
    for name, mod in mods.items():
        sys.modules[f"kbstub.{name}"] = mod
        setattr(pkg, name, mod)
    return pkg, mods, orig


def test_install_twice_with_options_on_a_stub_package():
    import sys

    pkg, mods, orig = _stub_kronblur()
    try:
        opts = kb.SolveOptions(dtype="float32", project=True)
        undo1 = kb.install(pkg, options=opts)
        assert callable(kb.install)  # the submodule import must not shadow the function
        undo2 = kb.install(pkg, options=kb.SolveOptions(dtype="float64"))
        pipe = mods["pipeline"]
        assert pipe.kron_apply is kb.kron_apply and mods["solvers"].kron_apply is kb.kron_apply
        assert pipe.decompose is kb.decompose and mods["kron"].decompose is kb.decompose
        assert pipe.estimate_lipschitz is kb.estimate_lipschitz
        assert pipe.sfista is not orig["sfista"] and mods["solvers"].sfista is not orig["sfista"]
        assert pipe.blur_direct is kb.blur_direct and mods["imaging"].blur_direct is kb.blur_direct
        # restore()'s vector-form closures are tagged for the device power iteration
        op = kb.decompose(random_psf(np.random.default_rng(1), 5), kb.BoundaryCondition.ZERO, s=2, shape=(8, 8))
        apply_vec, adjoint_vec = pipe._vec_ops(op)
        assert apply_vec._kb_power == (op, "vector", "float64")
        with pytest.raises(kb.ArgumentError):
            kb.install(pkg, options="float32")
        undo2()
        assert pipe.kron_apply is kb.kron_apply  # the first install is still in place
        undo1()
        for name, fn in orig.items():
            assert getattr(pipe, name) is fn
        assert mods["kron"].decompose is orig["decompose"] and pkg.sfista is orig["sfista"]
    finally:
        for name in [k for k in sys.modules if k == "kbstub" or k.startswith("kbstub.")]:
            del sys.modules[name]


def test_install_patches_every_by_name_binding(monkeypatch):
    from conftest import reference_module

    kronblur = reference_module()  # the reference, pip-installed into baseline/_ref by build()
    if kronblur is None:
        pytest.skip("reference not installed in baseline/_ref (run __graft_entry__.build() here)")
    from kronblur import pipeline, solvers

    orig = (solvers.sfista, pipeline.sfista, pipeline.estimate_lipschitz, pipeline.kron_apply)
    undo = kb.install(kronblur)
    try:
        assert solvers.sfista is not orig[0] and pipeline.sfista is solvers.sfista
        assert pipeline.estimate_lipschitz is kb.estimate_lipschitz
        assert pipeline.kron_apply is kb.kron_apply and solvers.kron_apply is kb.kron_apply
        assert kronblur.kron_apply_adjoint is kb.kron_apply_adjoint
        from kronblur import imaging, psf as ref_psf

        for mod in (kronblur, ref_psf, pipeline, imaging):
            assert mod.blur_direct is kb.blur_direct
        assert pipeline.decompose is kb.decompose and kronblur.kron.decompose is kb.decompose
        assert pipeline._vec_ops is not None and hasattr(pipeline._vec_ops(
            kb.decompose(random_psf(np.random.default_rng(2), 5), kb.BoundaryCondition.ZERO, s=1,
                         shape=(8, 8)))[0], "_kb_power")
    finally:
        undo()
    assert (solvers.sfista, pipeline.sfista, pipeline.estimate_lipschitz, pipeline.kron_apply) == orig


def test_product_never_imports_the_oracle_or_the_reference():
    """The oracle is test infrastructure and the reference is test-only data: nothing in the
    product package imports oracle/ or kronblur (other than errors.py reusing kronblur's error
    classes when kronblur is already importable, and dropin.py patching a module it is handed)."""
    import ast
    import glob

    pkg = os.path.join(ROOT, "paper_1901_00913_b200")
    for path in glob.glob(os.path.join(pkg, "*.py")):
        tree = ast.parse(open(path).read())
        for node in ast.walk(tree):
            names = []
            if isinstance(node, ast.Import):
                names = [a.name for a in node.names]
            elif isinstance(node, ast.ImportFrom):
                names = [node.module or ""]
            for name in names:
                assert not name.startswith("oracle"), (path, name)
                if name.startswith("kronblur"):
                    assert os.path.basename(path) == "errors.py", (path, name)
    # and the compute path fails loudly without the native library
    src = open(os.path.join(pkg, "device.py")).read()
    assert "no CPU fallback" in src
