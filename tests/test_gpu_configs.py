"""Per-config parity: every BASELINE configuration's PSF family, band width, rank, BC, lambda and
dtype, solved on the GPU and by the CPU oracle (oracle/kronblur_port.py) on the same seeded
inputs.

The oracle runs at sizes it finishes in seconds. cfg1 is at its full size; cfg2-cfg5 keep their
bands and ranks on smaller images. At the full cfg4/cfg5 sizes the checks are size-independent:
* the adjoint identity;
* fp32 against the fp64 GPU path.

Tolerances (north_star):
* fp64: relative Frobenius <= 1e-10;
* fp32: <= 1e-4, with PSNR against the truth within 0.01 dB of the oracle's.
"""

import numpy as np
import pytest

from conftest import cuda_ok

pytestmark = pytest.mark.gpu

if not cuda_ok():  # pragma: no cover - collected on CPU but skipped
    pytest.skip("needs a CUDA device", allow_module_level=True)

import torch  # noqa: E402

import paper_1901_00913_b200 as kb  # noqa: E402
from oracle import kronblur_port as port  # noqa: E402
from paper_1901_00913_b200 import workloads as W  # noqa: E402
from test_gpu_parity import rel  # noqa: E402


def psnr(x, ref):
    mse = float(np.mean((np.asarray(x, np.float64) - ref) ** 2))
    return 10.0 * np.log10(float(np.max(ref)) ** 2 / mse)


def solve_both(name, m, iters, dtype, seed=0, counts=(40, 20)):
    cfg = W.CONFIGS[name]
    X, psf, B = W.make_image_data(cfg, seed=seed, m=m, counts=counts, device="cuda")
    op = kb.decompose(psf, kb.BoundaryCondition(cfg.bc), s=cfg.r, shape=(m, m))
    if dtype == "float32":  # the oracle sees the fp32-rounded data
        B = B.astype(np.float32).astype(np.float64)
    L = kb.lipschitz(op, iters=20, seed=seed)
    run = kb.sfista(op, B, kb.SolveConfig(lam=cfg.lam, lipschitz=L, max_iter=iters, record_history=False),
                    options=kb.SolveOptions(dtype=dtype, project=True))
    want, _ = port.sfista(op, B, L, cfg.lam, iters, project=True)
    return X, run.x, want


@pytest.mark.parametrize("name,m,iters,dtype", [
    ("cfg1", 256, 100, "float64"),   # full size
    ("cfg2", 256, 60, "float64"),
    ("cfg2", 256, 60, "float32"),
    ("cfg4", 384, 20, "float32"),    # w = 255 band on a 384^2 image
    ("cfg5", 320, 20, "float32"),    # reflective w = 127 motion PSF, r = 10
])
def test_config_solve_matches_oracle(name, m, iters, dtype):
    X, got, want = solve_both(name, m, iters, dtype)
    if dtype == "float64":
        assert rel(got, want) <= 1e-10
    else:
        assert rel(got, want) <= 1e-4
        assert abs(psnr(got, X) - psnr(want, X)) <= 0.01
    assert np.all(got >= 0)


def test_cfg3_batch_matches_per_image_oracle():
    cfg = W.CONFIGS["cfg3"]
    m, nb, iters = 128, 6, 40
    ops, Bs, Xs = [], [], []
    for i in range(nb):
        X, psf, B = W.make_image_data(cfg, seed=0, index=i, m=m, counts=(20, 10), device="cuda")
        ops.append(kb.decompose(psf, kb.BoundaryCondition(cfg.bc), s=cfg.r, shape=(m, m)))
        Bs.append(B.astype(np.float32).astype(np.float64))
        Xs.append(X)
    Ls = np.array([kb.lipschitz(op, iters=20, seed=0) for op in ops])
    from paper_1901_00913_b200.device import DeviceOperator

    dev = DeviceOperator(ops, "float32")
    x, _ = kb.sfista_batch(dev, np.stack(Bs), Ls, cfg.lam, iters, options=kb.SolveOptions(project=True))
    for i in range(nb):
        want, _ = port.sfista(ops[i], Bs[i], Ls[i], cfg.lam, iters, project=True)
        assert rel(x[i], want) <= 1e-4
        assert abs(psnr(x[i], Xs[i]) - psnr(want, Xs[i])) <= 0.01


@pytest.mark.parametrize("name", ["cfg4", "cfg5"])
def test_full_size_operator_properties(name):
    # full BASELINE size: adjointness of the fp32 and fp64 operators, and fp32 == fp64 to 1e-5
    from paper_1901_00913_b200.device import DeviceOperator

    cfg = W.CONFIGS[name]
    m = cfg.m
    psf = W.make_psf(cfg)
    op = kb.decompose(psf, kb.BoundaryCondition(cfg.bc), s=cfg.r, shape=(m, m))
    g = torch.Generator(device="cuda").manual_seed(7)
    X = torch.rand((m, m), generator=g, device="cuda", dtype=torch.float64)
    Y = torch.rand((m, m), generator=g, device="cuda", dtype=torch.float64)
    d64 = DeviceOperator([op], "float64")
    AX = d64.apply(X)
    ATY = d64.apply(Y, adjoint=True)
    lhs = float(torch.sum(AX * Y))
    rhs = float(torch.sum(X * ATY))
    assert abs(lhs - rhs) <= 1e-11 * abs(lhs)
    d32 = DeviceOperator([op], "float32")
    AX32 = d32.apply(X.float()).double()
    assert float(torch.linalg.norm(AX32 - AX) / torch.linalg.norm(AX)) <= 1e-5
    ATY32 = d32.apply(Y.float(), adjoint=True).double()
    assert float(torch.linalg.norm(ATY32 - ATY) / torch.linalg.norm(ATY)) <= 1e-5
    del d64, d32
    torch.cuda.empty_cache()


def test_cfg3_style_batch_on_tensor_core_passes():
    """A batch large enough for the >= 8 chunks-per-SM rule (160 x 256^2, cfg3's w = 31 band) runs
    on the tcgen05 passes; sampled images match the per-image oracle at the fp32 tolerance."""
    from paper_1901_00913_b200.device import DeviceOperator

    cfg = W.CONFIGS["cfg3"]
    m, nb, iters = 256, 160, 30
    ops, Bs, Xs = [], [], []
    for i in range(nb):
        X, psf, B = W.make_image_data(cfg, seed=1, index=i, m=m, counts=(20, 10), device="cuda")
        ops.append(kb.decompose(psf, kb.BoundaryCondition(cfg.bc), s=cfg.r, shape=(m, m)))
        Bs.append(B.astype(np.float32).astype(np.float64))
        Xs.append(X)
    Ls = np.array([kb.lipschitz(op, iters=20, seed=0) for op in ops])
    dev = DeviceOperator(ops, "float32")
    B32 = torch.from_numpy(np.stack(Bs)).to("cuda", torch.float32)
    dev.time_passes(B32, B32, Ls, cfg.lam, reps=1)
    assert dev.last_engines() == ["tcgen05_tf32"] * 4
    x, _ = kb.sfista_batch(dev, np.stack(Bs), Ls, cfg.lam, iters, options=kb.SolveOptions(project=True))
    for i in (0, 77, nb - 1):
        want, _ = port.sfista(ops[i], Bs[i], Ls[i], cfg.lam, iters, project=True)
        assert rel(x[i], want) <= 1e-4
        assert abs(psnr(x[i], Xs[i]) - psnr(want, Xs[i])) <= 0.01
