"""GPU exact blur (kb_blur_direct, psf.py:170-193 blur_direct) against the reference's golden
vectors and the CPU oracle: BIT-EXACT (the kernel replays the reference's per-pixel sequence of
separately rounded fp64 products and sums)."""

import os

import numpy as np
import pytest

from conftest import GOLDEN, cuda_ok, random_psf

pytestmark = pytest.mark.gpu

if not cuda_ok():  # pragma: no cover - collected on CPU but skipped
    pytest.skip("needs a CUDA device", allow_module_level=True)

import torch  # noqa: E402

import paper_1901_00913_b200 as kb  # noqa: E402
from paper_1901_00913_b200.blur import blur_direct, blur_direct_batch  # noqa: E402
from oracle import kronblur_port as port  # noqa: E402

BCS = (kb.BoundaryCondition.ZERO, kb.BoundaryCondition.REFLECTIVE)


def test_golden_vectors_bit_exact():
    g = np.load(os.path.join(GOLDEN, "blur.npz"))
    for ci in range(int(g["ncases"])):
        psf = kb.Psf(g[f"b{ci}_psf"], tuple(int(v) for v in g[f"b{ci}_center"]))
        X = g[f"b{ci}_X"]
        for bc in BCS:
            got = blur_direct(psf, X, bc)
            assert got.dtype == np.float64 and got.shape == X.shape
            assert np.array_equal(got, g[f"b{ci}_{bc.value}_Y"]), (ci, bc)


@pytest.mark.parametrize("shape,psf_shape", [((97, 130), (41, 23)), ((256, 256), (31, 31)),
                                             ((70, 33), (70, 5)), ((5, 300), (5, 299))])
def test_random_against_oracle_bit_exact(rng, shape, psf_shape):
    psf = random_psf(rng, *psf_shape)
    X = rng.standard_normal(shape)
    for bc in BCS:
        assert np.array_equal(blur_direct(psf, X, bc), port.blur_direct(psf.values, psf.center, X, bc.value))


def test_sparse_psf_and_padded_psf_agree(rng):
    """Cropping all-zero borders (host) and skipping zero entries (kernel) reproduce the reference's
    np.nonzero loop: a pad_to'ed PSF gives the same image as the compact one, bit for bit."""
    vals = rng.random((9, 7)) + 0.05
    vals[2, :] = 0.0
    vals[:, 4] = 0.0
    vals /= vals.sum()
    psf = kb.Psf(vals, (3, 5))
    X = rng.standard_normal((48, 40))
    for bc in BCS:
        a = blur_direct(psf, X, bc)
        b = blur_direct(kb.pad_to(psf, 48, 40), X, bc)
        assert np.array_equal(a, b)
        assert np.array_equal(a, port.blur_direct(vals, (3, 5), X, bc.value))


def test_device_tensor_path_and_batch(rng):
    psfs = [random_psf(rng, 11, 11) for _ in range(3)]
    psfs = [kb.Psf(p.values, (6, 6)) for p in psfs]
    X = torch.from_numpy(rng.standard_normal((3, 64, 72))).cuda()
    for bc in BCS:
        batch = blur_direct_batch(psfs, X, bc)
        for k in range(3):
            one = blur_direct(psfs[k], X[k], bc)
            assert isinstance(one, torch.Tensor) and one.is_cuda
            assert torch.equal(batch[k], one)
            assert np.array_equal(one.cpu().numpy(),
                                  port.blur_direct(psfs[k].values, (6, 6), X[k].cpu().numpy(), bc.value))


def test_errors_match_reference(rng):
    psf = random_psf(rng, 9, 9)
    with pytest.raises(kb.ArgumentError, match="larger than image"):
        blur_direct(psf, np.zeros((8, 20)), BCS[0])
    with pytest.raises(kb.ArgumentError, match="image must be 2-D"):
        blur_direct(psf, np.zeros((4, 20, 20)), BCS[0])


@pytest.mark.parametrize("cfg_name", ["cfg4", "cfg5"])
def test_full_size_sampled_pixels_bit_exact(cfg_name):
    """BASELINE full sizes (4096², 255² Moffat; 16384², 127² motion PSF): the whole image would take
    hours in numpy, so sampled pixels (corners, edges, interior) are checked against the oracle's
    per-pixel restatement of the same sequence."""
    from paper_1901_00913_b200 import workloads as W

    cfg = W.CONFIGS[cfg_name]
    psf = W.make_psf(cfg)
    m = cfg.m
    gen = torch.Generator(device="cuda").manual_seed(7)
    X = torch.rand((m, m), device="cuda", dtype=torch.float64, generator=gen)
    bc = kb.BoundaryCondition(cfg.bc)
    Y = blur_direct(psf, X, bc)
    rng = np.random.default_rng(11)
    pts = [(0, 0), (0, m - 1), (m - 1, 0), (m - 1, m - 1), (m // 2, 3), (5, m // 2)]
    pts += [tuple(int(v) for v in rng.integers(0, m, 2)) for _ in range(6)]
    rows, _ = psf.values.shape
    l = psf.center[0]
    Xh = np.zeros((m, m))  # calloc: only the copied rows are committed
    for i, j in pts:
        # pixel i reads input rows i + l - 1 - a (a < rows), folded once at the edges
        need = sorted({t if 0 <= t < m else (-1 - t if t < 0 else 2 * m - 1 - t)
                       for t in range(i + l - rows, i + l)} & set(range(m)))
        Xh[need] = X.index_select(0, torch.tensor(need, device="cuda")).cpu().numpy()
        want = port.blur_direct_pixel(psf.values, psf.center, Xh, cfg.bc, i, j)
        assert float(Y[i, j]) == want, (cfg_name, i, j)
