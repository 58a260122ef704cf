"""fp32 GPU path against the CPU oracle (oracle/kronblur_port.py).

Shapes with both extents a multiple of 4 run the persistent TMA + FFMA kernels (kb_ffma.cuh);
the others run the generic tiled kernels. Tolerances (north_star): fp32 relative Frobenius
<= 1e-4 and PSNR within 0.01 dB of the fp64 oracle; integer-valued inputs small enough to be
exact in fp32 are compared bit for bit.
"""

import numpy as np
import pytest

from conftest import cuda_ok, random_psf

pytestmark = pytest.mark.gpu

if not cuda_ok():  # pragma: no cover - collected on CPU but skipped
    pytest.skip("needs a CUDA device", allow_module_level=True)

import torch  # noqa: E402

import paper_1901_00913_b200 as kb  # noqa: E402
from oracle import kronblur_port as port  # noqa: E402
from test_gpu_parity import int_operator, rel  # noqa: E402

ZERO = kb.BoundaryCondition.ZERO
REFL = kb.BoundaryCondition.REFLECTIVE


def psnr(x, ref):
    mse = float(np.mean((np.asarray(x, np.float64) - ref) ** 2))
    return 10.0 * np.log10(float(np.max(ref)) ** 2 / mse)


@pytest.mark.parametrize("bc", ["zero", "reflective"])
@pytest.mark.parametrize("shape,r,ha,hb", [((64, 96), 3, 6, 9), ((132, 260), 5, 31, 20),
                                            ((36, 40), 2, 17, 3), ((33, 40), 3, 6, 6),
                                            ((8, 8), 1, 4, 4), ((300, 4), 2, 11, 2)])
def test_integer_apply_bit_exact_fp32(bc, shape, r, ha, hb, rng):
    m, n = shape
    op = int_operator(rng, m, n, r, bc, min(ha, m - 1), min(hb, n - 1), lo=-3, hi=3)
    X = rng.integers(-4, 5, size=(m, n)).astype(float)
    want = port.dense_kron_apply(op, X)
    wantT = port.dense_kron_apply(op, X, adjoint=True)
    assert np.max(np.abs(want)) < 2**24 and np.max(np.abs(wantT)) < 2**24
    assert np.array_equal(kb.kron_apply(op, X, dtype="float32"), want)
    assert np.array_equal(kb.kron_apply_adjoint(op, X, dtype="float32"), wantT)


@pytest.mark.parametrize("bc", [ZERO, REFL])
@pytest.mark.parametrize("m,size,s", [(64, 9, 3), (256, 31, 3), (200, 15, 4), (96, 63, 5), (98, 21, 3)])
def test_apply_matches_oracle_fp32(bc, m, size, s, rng):
    psf = random_psf(rng, size)
    op = kb.decompose(psf, bc, s=s, shape=(m, m))
    pop = port.PortOperator(op)
    X = rng.standard_normal((m, m))
    assert rel(kb.kron_apply(op, X, dtype="float32"), port.kron_apply(pop, X)) <= 1e-5
    assert rel(kb.kron_apply_adjoint(op, X, dtype="float32"), port.kron_apply_adjoint(pop, X)) <= 1e-5


@pytest.mark.parametrize("exact", [False, True])
@pytest.mark.parametrize("name", ["cfg1", "cfg2", "cfg5"])
def test_symmetric_generators_fp32(name, exact, monkeypatch):
    from paper_1901_00913_b200 import workloads as W
    from paper_1901_00913_b200.device import DeviceOperator

    cfg = W.CONFIGS[name]
    m = (3 * cfg.w + 7) // 4 * 4
    op = kb.decompose(W.make_psf(cfg), REFL, s=cfg.r, shape=(m, m))
    if exact:
        monkeypatch.setenv("KB_EXACT_FOLD", "1")
    dev = DeviceOperator([op], "float32")
    assert dev.info()["sym_a"] == (0 if exact else 1)
    X = np.random.default_rng(5).standard_normal((m, m))
    t = torch.from_numpy(X).cuda().float()
    pop = port.PortOperator(op)
    assert rel(dev.apply(t, adjoint=True).double().cpu().numpy(), port.kron_apply_adjoint(pop, X)) <= 1e-5
    assert rel(dev.apply(t).double().cpu().numpy(), port.kron_apply(pop, X)) <= 1e-5


@pytest.mark.parametrize("bc", [ZERO, REFL])
def test_sfista_fp32_matches_oracle(bc, rng):
    from paper_1901_00913_b200 import workloads as W

    cfg = W.CONFIGS["cfg2"]
    m = 256
    X, psf, B = W.make_image_data(cfg, seed=1, m=m, counts=(40, 20))
    op = kb.decompose(psf, bc, s=cfg.r, shape=(m, m))
    L = 1.0
    want, _ = port.sfista(op, B, L, cfg.lam, 60, project=True)
    run = kb.sfista(op, B, kb.SolveConfig(lam=cfg.lam, lipschitz=L, max_iter=60, record_history=False),
                    options=kb.SolveOptions(dtype="float32", project=True))
    assert rel(run.x, want) <= 1e-4
    assert abs(psnr(run.x, X) - psnr(want, X)) <= 0.01


def test_power_iteration_fp32(rng):
    psf = random_psf(rng, 9)
    m = 64
    op = kb.decompose(psf, REFL, s=3, shape=(m, m))
    pop = port.PortOperator(op)
    want = port.estimate_lipschitz(lambda v: port.kron_apply(pop, v),
                                   lambda v: port.kron_apply_adjoint(pop, v), (m, m), 40, 2)
    got = kb.lipschitz(op, iters=40, seed=2, dtype="float32")
    assert abs(got - want) <= 1e-5 * want


def test_batched_solve_fp32(rng):
    from paper_1901_00913_b200.device import DeviceOperator

    ops, Bs, Ls = [], [], []
    for i in range(3):
        op = kb.decompose(random_psf(rng, 7), REFL, s=2, shape=(64, 64))
        ops.append(op)
        Bs.append(rng.random((64, 64)))
        Ls.append(1.0 + 0.1 * i)
    dev = DeviceOperator(ops, "float32")
    x, _ = kb.sfista_batch(dev, np.stack(Bs), np.array(Ls), 0.02, 30, options=kb.SolveOptions(project=True))
    for i in range(3):
        want, _ = port.sfista(ops[i], Bs[i], Ls[i], 0.02, 30, project=True)
        assert rel(x[i], want) <= 1e-4
