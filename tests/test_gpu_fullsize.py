"""Full-size parity of every BASELINE config, on the default engine policy.

Each case names its config, size and iteration count. The GPU side runs exactly what bench.py
times: the seeded BASELINE data generated on the device, the public ``sfista`` / ``sfista_batch``
with the default engine policy (asserted through ``last_engines``), projection on. Two checkers:

* full-length fixtures (tests/golden/full_*.npz) computed offline by the C restatement of the
  reference hot path (oracle/kb_oracle.c, pinned to the reference by tests/test_oracle_c.py;
  generator: tests/golden/make_fullsize.py). They hold L, a fingerprint of B, every row norm,
  sampled full rows and the PSNR of the oracle's solution;
* live oracle runs on this host at full size for the first iterations (cfg2: all 200; cfg4: 3;
  cfg5: 2), plus the numpy port of the reference's own FFT path for cfg2's first iterations.

Tolerances (north_star): fp64 relative Frobenius <= 1e-10; fp32 <= 1e-4 and PSNR against the
ground truth within 0.01 dB of the oracle's (fp32 runs feed the oracle the fp32-rounded data
and taps).
"""

import os

import numpy as np
import pytest

from conftest import GOLDEN, cuda_ok

pytestmark = pytest.mark.gpu

if not cuda_ok():  # pragma: no cover - collected on CPU but skipped
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1901_00913_b200 as kb  # noqa: E402
from oracle import kb_oracle as C  # noqa: E402
from oracle import kronblur_port as port  # noqa: E402
from paper_1901_00913_b200 import workloads as W  # noqa: E402
from paper_1901_00913_b200.device import DeviceOperator, device_operator  # noqa: E402

TOL = {"float64": 1e-10, "float32": 1e-4}
# default-policy engines of the four phases (split fwd, sum fwd, split adj, sum adj) at full size
EXPECT = {
    ("cfg2", "float64"): ["dmma"] * 4,
    ("cfg3", "float32"): ["tcgen05_tf32"] * 4,
    ("cfg4", "float32"): ["tcgen05_tf32"] * 4,
    ("cfg5", "float32"): ["tcgen05_tf32"] * 4,
}


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a, np.float64) - b) / np.linalg.norm(b))


def psnr(x, truth):
    return 10.0 * np.log10(1.0 / float(np.mean((np.asarray(x, np.float64) - truth) ** 2)))


def fixture(case):
    path = os.path.join(GOLDEN, f"full_{case}.npz")
    if not os.path.exists(path):
        pytest.fail(f"missing fixture {path} (tests/golden/make_fullsize.py)")
    return np.load(path)


def check_b(B, f, pre=""):
    """The regenerated data B is the fixture's (phantom painting is exact and blur_direct is
    bit-identical on both sides; only the noise scale's last bits may depend on BLAS)."""
    got = B.ravel()[f[pre + "b_idx"]]
    assert np.max(np.abs(got - f[pre + "b_vals"])) <= 1e-12 * np.max(np.abs(f[pre + "b_vals"]))
    assert float(B.sum()) == pytest.approx(float(f[pre + "b_sum"]), rel=1e-12)


def check_x(x, X, f, dtype, pre=""):
    tol = TOL[dtype]
    rows = f[pre + "rows_idx"]
    assert rel(x[rows], f[pre + "rows"].astype(np.float64)) <= tol
    assert rel(np.linalg.norm(x, axis=1), f[pre + "row_norms"]) <= tol
    assert float(np.linalg.norm(x)) == pytest.approx(float(f[pre + "fro"]), rel=tol)
    if dtype == "float32":
        assert abs(psnr(x, X) - float(f[pre + "psnr"])) <= 0.01
    assert np.all(x >= 0)


def solve(op, B, L, cfg, dtype, iters):
    run = kb.sfista(op, B, kb.SolveConfig(lam=cfg.lam, lipschitz=L, max_iter=iters, record_history=False),
                    options=kb.SolveOptions(dtype=dtype, project=True))
    return run.x, device_operator(op, dtype).last_engines()


@pytest.mark.parametrize("case", ["cfg2_float64", "cfg2_float32", "cfg4_float32", "cfg5_float32"])
def test_full_length_solve_matches_fixture(case):
    """cfg2 1024^2 x 200 it (fp64, fp32), cfg4 4096^2 x 300 it, cfg5 16384^2 x 100 it."""
    f = fixture(case)
    name, dtype = str(f["config"]), str(f["dtype"])
    cfg = W.CONFIGS[name]
    X, psf, B = W.make_image_data(cfg, seed=0, device="cuda")
    check_b(B, f)
    op = kb.decompose(psf, kb.BoundaryCondition(cfg.bc), s=cfg.r, shape=(cfg.m, cfg.m))
    x, engines = solve(op, B, float(f["L"]), cfg, dtype, int(f["iters"]))
    if (name, dtype) in EXPECT:
        assert engines == EXPECT[(name, dtype)], engines
    assert "generic" not in engines and "ffma" not in engines, engines
    check_x(x, X, f, dtype)


def test_cfg3_full_batch_matches_fixture():
    """cfg3: the whole 512-image batch (512 x 512^2, r=4, 100 it) in one batched solve on the
    default tcgen05 policy; 8 sampled images checked against the oracle's full-length solves."""
    f = fixture("cfg3_float32")
    cfg = W.CONFIGS["cfg3"]
    sampled = [int(i) for i in f["images"]]
    ops, Bs, Xs = [], [], {}
    for i in range(cfg.batch):
        X, psf, B = W.make_image_data(cfg, seed=0, index=i, device="cuda")
        if i in sampled:
            check_b(B, f, f"i{i}_")
            Xs[i] = X
        ops.append(kb.decompose(psf, kb.BoundaryCondition(cfg.bc), s=cfg.r, shape=(cfg.m, cfg.m)))
        Bs.append(B)
    L = np.full(cfg.batch, 1.1)  # unsampled images: any L above their Lipschitz constant
    for i in sampled:
        L[i] = float(f[f"i{i}_L"])
    dev = DeviceOperator(ops, "float32")
    x, _ = kb.sfista_batch(dev, np.stack(Bs), L, cfg.lam, cfg.iters,
                           options=kb.SolveOptions(dtype="float32", project=True))
    assert dev.last_engines() == EXPECT[("cfg3", "float32")], dev.last_engines()
    for i in sampled:
        check_x(x[i], Xs[i], f, "float32", f"i{i}_")


@pytest.mark.parametrize("name,dtype,iters", [
    ("cfg2", "float64", 200),
    ("cfg2", "float32", 200),
    ("cfg4", "float32", 3),
    ("cfg5", "float32", 2),
])
def test_full_size_against_live_oracle(name, dtype, iters):
    """The first `iters` iterations at full size against the C oracle run here and now (and,
    for cfg2, the first 5 iterations against the numpy port of the reference's FFT path)."""
    cfg = W.CONFIGS[name]
    X, psf, B = W.make_image_data(cfg, seed=0, device="cuda")
    op = kb.decompose(psf, kb.BoundaryCondition(cfg.bc), s=cfg.r, shape=(cfg.m, cfg.m))
    L = kb.lipschitz(op, iters=50, seed=0)
    Bin = B.astype(np.float32).astype(np.float64) if dtype == "float32" else B
    _, beta = kb.momentum_table(iters)
    want = C.sfista(C.OracleOp(op, dtype), Bin, L, cfg.lam, iters, beta, project=True)
    got, engines = solve(op, Bin, L, cfg, dtype, iters)
    assert "generic" not in engines, engines
    assert rel(got, want) <= TOL[dtype]
    if name == "cfg2":
        port.set_threads(os.cpu_count() or 1)
        ref5, _ = port.sfista(op, Bin, L, cfg.lam, 5, project=True)
        got5, _ = solve(op, Bin, L, cfg, dtype, 5)
        assert rel(got5, ref5) <= TOL[dtype]


def test_cfg1_against_the_references_own_solution():
    """cfg1 (256^2 fp64, zero BC, w=31, r=3, lam=0.02, 100 it) with the reference's own factors,
    data and L (tests/golden/cfg1.npz, written by running kronblur itself): the GPU solve -- the
    whole-solve persistent kernel at this size -- reproduces the reference's projected solution
    and, without projection, kronblur.sfista's own x."""
    g = np.load(os.path.join(GOLDEN, "cfg1.npz"))
    terms = tuple(kb.KronTerm(sigma=1.0, H=kb.toep(g["H_c"][i], int(g["H_j"])), K=kb.toep(g["K_c"][i], int(g["K_j"])))
                  for i in range(g["H_c"].shape[0]))
    op = kb.KronOperator(terms=terms, shape=(256, 256), bc=kb.BoundaryCondition.ZERO, sigma=np.ones(len(terms)),
                         s=len(terms), rank=len(terms), eps=0.0)
    cfg = kb.SolveConfig(lam=0.02, lipschitz=float(g["L"]), max_iter=100, record_history=False)
    for project, want in ((True, g["x_proj"]), (False, g["x_sfista"])):
        run = kb.sfista(op, g["B"], cfg, options=kb.SolveOptions(dtype="float64", project=project))
        assert rel(run.x, want) <= 1e-10
    assert device_operator(op, "float64").last_engines() == ["persist_f64"] * 4
