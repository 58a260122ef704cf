"""Row-block device kernels (kb_block_residual / kb_block_update / kb_apply_block) on one GPU.

The ranks of a row-sharded solve are emulated sequentially in one process: each block gets its
halo rows copied from the neighbouring blocks (what exchange_halos does over NCCL), and the
assembled result must equal the single-device solve. Nothing here waits on another launch.
"""

import numpy as np
import pytest

from conftest import cuda_ok, random_psf

pytestmark = pytest.mark.gpu

if not cuda_ok():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import torch  # noqa: E402

import paper_1901_00913_b200 as kb  # noqa: E402
from paper_1901_00913_b200 import shard  # noqa: E402
from oracle import kronblur_port as port  # noqa: E402


def emulate_row_blocks(op, B, L, lam, iters, world, dtype="float64", split=False):
    m, n = op.shape
    h = shard.halo_rows(op)
    plans = [shard.BlockPlan(m=m, n=n, world=world, rank=r, h=h) for r in range(world)]
    backs = [shard.DeviceBlockBackend(op, p, dtype) for p in plans]
    td = torch.float64 if dtype == "float64" else torch.float32
    Yh = [torch.zeros((p.rows + 2 * h, n), dtype=td, device="cuda") for p in plans]
    Rh = [torch.zeros_like(y) for y in Yh]
    X = [torch.zeros((p.rows, n), dtype=td, device="cuda") for p in plans]
    Bl = [torch.from_numpy(B[p.g0:p.g0 + p.rows].copy()).to("cuda", td) for p in plans]
    flag = torch.full((1,), 2**31 - 1, dtype=torch.int32, device="cuda")
    _, beta = kb.momentum_table(iters)

    def ranges(p):
        if not split:
            return [(0, p.rows)]
        return [(h, p.rows - h), (0, h), (p.rows - h, p.rows)]

    def exchange(bufs):
        for r, p in enumerate(plans):
            if p.prev is not None:
                bufs[r][0:h] = bufs[r - 1][plans[r - 1].rows:plans[r - 1].rows + h]
            if p.next is not None:
                bufs[r][h + p.rows:2 * h + p.rows] = bufs[r + 1][h:2 * h]

    for k in range(1, iters + 1):
        exchange(Yh)
        for r in range(world):
            for r0, r1 in ranges(plans[r]):  # split=True: the overlap path's interior + edge strips
                backs[r].residual(Yh[r], Bl[r], Rh[r], r0, r1)
        exchange(Rh)
        for r in range(world):
            for r0, r1 in ranges(plans[r]):
                backs[r].update(Rh[r], X[r], Yh[r], beta[k - 1], k, L, lam, True, flag, r0, r1)
    torch.cuda.synchronize()
    assert int(flag.item()) > iters
    return torch.cat(X).double().cpu().numpy()


@pytest.mark.parametrize("bc", ["zero", "reflective"])
@pytest.mark.parametrize("world", [2, 3])
def test_row_blocks_match_single_device(bc, world, rng):
    psf = random_psf(rng, 9)
    op = kb.decompose(psf, kb.BoundaryCondition(bc), s=3, shape=(90, 90))
    B = rng.random((90, 90))
    got = emulate_row_blocks(op, B, 1.4, 0.03, 20, world)
    want, _ = port.sfista(op, B, 1.4, 0.03, 20, project=True)
    np.testing.assert_allclose(got, want, rtol=0, atol=1e-10 * np.abs(want).max())


def test_row_blocks_symmetric_psf_fp32():
    from paper_1901_00913_b200 import workloads as W

    cfg = W.CONFIGS["cfg5"]
    m = 300
    op = kb.decompose(W.make_psf(cfg), kb.BoundaryCondition("reflective"), s=4, shape=(m, m))
    B = np.random.default_rng(2).random((m, m))
    got = emulate_row_blocks(op, B, 1.1, 0.01, 10, 2, dtype="float32")
    want, _ = port.sfista(op, B, 1.1, 0.01, 10, project=True)
    assert np.linalg.norm(got - want) / np.linalg.norm(want) <= 1e-5


def test_apply_block_matches_full(rng):
    from paper_1901_00913_b200 import device as D

    psf = random_psf(rng, 7)
    op = kb.decompose(psf, kb.BoundaryCondition.REFLECTIVE, s=2, shape=(64, 64))
    X = rng.standard_normal((64, 64))
    full = port.kron_apply(port.PortOperator(op), X)
    fullT = port.kron_apply_adjoint(port.PortOperator(op), X)
    h = shard.halo_rows(op)
    g0, rows = 20, 24
    be = shard.DeviceBlockBackend(op, shard.BlockPlan(m=64, n=64, world=1, rank=0, h=h))
    dev = D.DeviceOperator([shard._LocalShape(op, rows)], "float64")
    Xh = torch.from_numpy(X[g0 - h:g0 + rows + h].copy()).cuda()
    out = torch.empty((rows, 64), dtype=torch.float64, device="cuda")
    for adj, want in ((0, full), (1, fullT)):
        rc = D.load_library().kb_apply_block(dev._handle, adj, D._ptr(Xh[h:]), D._ptr(out),
                                             D._ptr(dev.work), g0, 64, h, h, D._stream_handle())
        D._check(rc, "kb_apply_block")
        np.testing.assert_allclose(out.cpu().numpy(), want[g0:g0 + rows], rtol=0, atol=1e-12)
    del be


def test_batch_shard_partition_covers_all_images(rng):
    ops, Bs = [], []
    for _ in range(5):
        ops.append(kb.decompose(random_psf(rng, 5), kb.BoundaryCondition.ZERO, s=2, shape=(32, 32)))
        Bs.append(rng.random((32, 32)))
    Bs = np.stack(Bs)
    L = np.full(5, 1.2)
    xs = {}
    for rank in range(2):
        start, x, _ = shard.solve_batch_shard(ops, Bs, L, 0.02, 15, rank, 2,
                                              options=kb.SolveOptions(dtype="float64", project=True))
        for i in range(x.shape[0]):
            xs[start + i] = x[i]
    assert sorted(xs) == list(range(5))
    for i in range(5):
        want, _ = port.sfista(ops[i], Bs[i], 1.2, 0.02, 15, project=True)
        np.testing.assert_allclose(xs[i], want, rtol=0, atol=1e-10 * np.abs(want).max())


@pytest.mark.parametrize("bc", ["zero", "reflective"])
@pytest.mark.parametrize("dtype", ["float64", "float32"])
def test_overlap_sub_ranges_match_whole_blocks(bc, dtype, rng):
    """The overlap schedule computes each block as interior rows [h, rows-h) then the two h-row
    edge strips; the result must equal the whole-block computation."""
    psf = random_psf(rng, 11)
    op = kb.decompose(psf, kb.BoundaryCondition(bc), s=3, shape=(120, 120))
    B = rng.random((120, 120))
    whole = emulate_row_blocks(op, B, 1.4, 0.03, 12, 2, dtype)
    split = emulate_row_blocks(op, B, 1.4, 0.03, 12, 2, dtype, split=True)
    if dtype == "float64":
        np.testing.assert_allclose(split, whole, rtol=0, atol=1e-12 * np.abs(whole).max())
    else:  # thin strips may take other fp32 kernels (other summation order): fp32 rounding only
        assert np.linalg.norm(split - whole) / np.linalg.norm(whole) <= 2e-6


def test_single_rank_history_and_power_match_unsharded(rng):
    """world = 1: solve_row_blocks with record_history (device block norms, kb_resid_norms) and
    the sharded power iteration (kb_apply_block, kb_inner2) reproduce sfista's history and
    estimate_lipschitz."""
    from paper_1901_00913_b200.solvers import _start_vector

    psf = random_psf(rng, 9)
    op = kb.decompose(psf, kb.BoundaryCondition.REFLECTIVE, s=3, shape=(64, 64))
    B = rng.random((64, 64))
    plan = shard.BlockPlan(m=64, n=64, world=1, rank=0, h=shard.halo_rows(op))
    be = shard.DeviceBlockBackend(op, plan, "float64")
    L = shard.power_iter_row_blocks(be, plan, torch.from_numpy(_start_vector(4, 64, 64, "matrix")).cuda(), 50)
    assert L == pytest.approx(kb.lipschitz(op, iters=50, seed=4), rel=1e-12)
    X, hist = shard.solve_row_blocks(be, plan, torch.from_numpy(B).cuda(), L, 0.03, 15, project=True,
                                     record_history=True)
    run = kb.sfista(op, B, kb.SolveConfig(lam=0.03, lipschitz=L, max_iter=15, record_history=True),
                    options=kb.SolveOptions(dtype="float64", project=True))
    assert len(hist) == len(run.history) == 15
    for h, r in zip(hist, run.history):
        assert h["objective"] == pytest.approx(r.objective, rel=1e-11)
    np.testing.assert_allclose(X.cpu().numpy(), run.x, rtol=0, atol=1e-12)


@pytest.mark.parametrize("dtype", ["float64", "float32"])
def test_l2_blocked_schedule_is_bit_identical(dtype, monkeypatch, rng):
    """The opt-in L2-blocked schedule (KB_L2_STRIP rows per strip / KB_L2_GROUP images per group,
    kb_capi.cu sfista_blocked) runs the same kernels on pieces: fp64 results are bit-identical to
    the whole-plane schedule, fp32 ones agree to fp32 rounding."""
    from paper_1901_00913_b200.device import INT_MAX, DeviceOperator, device_operator

    psf = random_psf(rng, 15)
    op = kb.decompose(psf, kb.BoundaryCondition.REFLECTIVE, s=4, shape=(1024, 1024))
    B = torch.from_numpy(rng.random((1024, 1024))).cuda()
    dev = device_operator(op, dtype)
    _, beta = kb.momentum_table(6)
    outs = {}
    for strip in ("0", "128", "256"):
        monkeypatch.setenv("KB_L2_STRIP", strip)
        X, Y = torch.zeros_like(B, dtype=dev.tdtype), torch.zeros_like(B, dtype=dev.tdtype)
        flag = torch.full((1,), INT_MAX, dtype=torch.int32, device="cuda")
        dev.sfista_run(B.to(dev.tdtype), X, Y, beta, 0, 6, 1.2, 0.02, True, flag)
        outs[strip] = X.cpu()
    if dtype == "float64":
        assert torch.equal(outs["0"], outs["128"]) and torch.equal(outs["0"], outs["256"])
    else:  # fp32 tiling of a strip may reorder the 3xTF32 K-step sums: fp32 rounding only
        for k in ("128", "256"):
            assert float((outs[k] - outs["0"]).norm() / outs["0"].norm()) <= 1e-6
    ops = [kb.decompose(random_psf(rng, 7), kb.BoundaryCondition.ZERO, s=2, shape=(128, 128)) for _ in range(7)]
    devb = DeviceOperator(ops, dtype)
    Bb = torch.from_numpy(rng.random((7, 128, 128))).cuda().to(devb.tdtype)
    Ls = np.linspace(1.1, 1.3, 7)
    res = {}
    for group in ("0", "3"):
        monkeypatch.setenv("KB_L2_GROUP", group)
        X, Y = torch.zeros_like(Bb), torch.zeros_like(Bb)
        flag = torch.full((1,), INT_MAX, dtype=torch.int32, device="cuda")
        devb.sfista_run(Bb, X, Y, beta, 0, 6, Ls, 0.02, True, flag)
        res[group] = X.cpu()
    if dtype == "float64":
        assert torch.equal(res["0"], res["3"])
    else:
        assert float((res["3"] - res["0"]).norm() / res["0"].norm()) <= 1e-6


def test_row_blocks_of_the_transposed_image_match(rng):
    """The sharded solve in the axis-swapped frame (bench.py run_row_blocks with prefer_swap):
    row blocks of B^T with H and K swapped give x^T of the ordinary solve."""
    psf = random_psf(rng, 11)
    op = kb.decompose(psf, kb.BoundaryCondition.REFLECTIVE, s=3, shape=(96, 96))
    B = rng.random((96, 96))
    got = emulate_row_blocks(shard.swapped(op), np.ascontiguousarray(B.T), 1.3, 0.02, 15, 2)
    want, _ = port.sfista(op, B, 1.3, 0.02, 15, project=True)
    np.testing.assert_allclose(got.T, want, rtol=0, atol=1e-10 * np.abs(want).max())
