"""Multi-rank plumbing of the sharded solvers on CPU (gloo, world_size 2).

The row-block solver's partition, halo exchange and global-edge handling are checked with a dense
CPU backend (the oracle's materialised factors restricted to the block rows and halo columns) in
place of the device kernels; the device kernels' own block logic is checked on one GPU in
test_gpu_blocks.py.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import ROOT, random_psf

import paper_1901_00913_b200 as kb
from paper_1901_00913_b200 import shard
from oracle import kronblur_port as port


class DenseBlockBackend:
    """The backend interface of shard.DeviceBlockBackend from dense factors (the oracle's
    materialised factors restricted to the block rows and halo columns): R = A Y - B and the
    projected FISTA update on local rows [r0, r1), block applies and the local reductions."""

    def __init__(self, op, plan):
        self.plan = plan
        self.Ha = [port.dense_factor(t.H) for t in op.terms]
        self.Kb = [port.dense_factor(t.K) for t in op.terms]

    def _cols(self):
        p = self.plan
        return slice(p.g0 - p.hlo, p.g0 + p.rows + p.hhi)

    def _halo(self, buf):
        p = self.plan
        return buf[p.h - p.hlo: p.h + p.rows + p.hhi].numpy()

    def residual(self, Yh, B, R, r0=0, r1=None):
        p = self.plan
        r1 = p.rows if r1 is None else r1
        rows, cols = slice(p.g0 + r0, p.g0 + r1), self._cols()
        Y = self._halo(Yh)
        acc = sum(Ha[rows, cols] @ Y @ Kb.T for Ha, Kb in zip(self.Ha, self.Kb))
        R[p.h + r0:p.h + r1] = torch.from_numpy(acc - B[r0:r1].numpy())

    def update(self, Rh, X, Yh, beta, k, L, lam, project, flag, r0=0, r1=None, norms=None):
        p = self.plan
        r1 = p.rows if r1 is None else r1
        rows, cols = slice(p.g0 + r0, p.g0 + r1), self._cols()
        Rm = self._halo(Rh)
        G = sum(Ha.T[rows, cols] @ Rm @ Kb for Ha, Kb in zip(self.Ha, self.Kb))
        y = Yh[p.h + r0:p.h + r1].numpy()
        xp = X[r0:r1].numpy().copy()
        x = (L * y - G) / (L + lam**2)
        if project:
            x = np.maximum(x, 0.0)
        X[r0:r1] = torch.from_numpy(x)
        Yh[p.h + r0:p.h + r1] = torch.from_numpy(x + beta * (x - xp))
        if norms is not None:
            norms[0] = float(np.sum((x - xp) ** 2))
            norms[1] = float(np.sum(xp ** 2))
            norms[2] = float(np.sum(x ** 2))

    def apply(self, Xh, out, adjoint=False):
        p = self.plan
        rows, cols = slice(p.g0, p.g0 + p.rows), self._cols()
        Xm = self._halo(Xh)
        if adjoint:
            acc = sum(Ha.T[rows, cols] @ Xm @ Kb for Ha, Kb in zip(self.Ha, self.Kb))
        else:
            acc = sum(Ha[rows, cols] @ Xm @ Kb.T for Ha, Kb in zip(self.Ha, self.Kb))
        out[:] = torch.from_numpy(acc)

    def resid2(self, AX, B, out2):
        out2[0] = float(np.sum((AX.numpy() - B.numpy()) ** 2))

    def inner2(self, a, b, out2):
        out2[0] = float(np.sum(a.numpy() * b.numpy()))
        out2[1] = float(np.sum(b.numpy() ** 2))


def _problem(bc):
    rng = np.random.default_rng(11)
    psf = random_psf(rng, 7)
    op = kb.decompose(psf, kb.BoundaryCondition(bc), s=3, shape=(26, 26))
    B = rng.random((26, 26))
    return op, B


def _worker(rank, world, port_no, bc, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port_no)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        op, B = _problem(bc)
        plan = shard.BlockPlan(m=26, n=26, world=world, rank=rank, h=shard.halo_rows(op))
        backend = DenseBlockBackend(op, plan)
        Bl = torch.from_numpy(B[plan.g0:plan.g0 + plan.rows].copy())
        X = shard.solve_row_blocks(backend, plan, Bl, 1.3, 0.05, 25, project=True)
        parts = [torch.zeros((r, 26), dtype=torch.float64) for _, r in plan.parts]
        dist.all_gather(parts, X)
        if rank == 0:
            out.put(torch.cat(parts).numpy())
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("bc", ["zero", "reflective"])
def test_row_block_solver_world2_matches_single(bc):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port_no = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port_no, bc, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
    codes = [p.exitcode for p in procs]
    for p in procs:
        if p.is_alive():
            p.kill()
    assert codes == [0, 0], codes
    got = q.get(timeout=10)
    op, B = _problem(bc)
    want, _ = port.sfista(op, B, 1.3, 0.05, 25, project=True)
    np.testing.assert_allclose(got, want, rtol=0, atol=1e-12 * np.abs(want).max())


def test_partitions():
    assert shard.row_partition(10, 3) == [(0, 4), (4, 3), (7, 3)]
    assert shard.batch_partition(5, 2) == [(0, 3), (3, 2)]
    assert shard.batch_partition(1, 3) == [(0, 1), (1, 0), (1, 0)]
    p = shard.BlockPlan(m=20, n=8, world=3, rank=1, h=2)
    assert (p.g0, p.rows, p.prev, p.next, p.hlo, p.hhi) == (7, 7, 0, 2, 2, 2)
    p0 = shard.BlockPlan(m=20, n=8, world=3, rank=0, h=2)
    assert (p0.hlo, p0.hhi) == (0, 2)
    with pytest.raises(kb.ArgumentError):
        shard.BlockPlan(m=6, n=8, world=3, rank=0, h=3)
    with pytest.raises(kb.ArgumentError):
        shard.row_partition(2, 3)


def _run_world2(target, *args):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port_no = _free_port()
    procs = [ctx.Process(target=target, args=(r, 2, port_no, q) + args) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=180)
    codes = [p.exitcode for p in procs]
    for p in procs:
        if p.is_alive():
            p.kill()
    assert codes == [0, 0], codes
    return q.get(timeout=10)


def _init(rank, world, port_no):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port_no)
    dist.init_process_group("gloo", rank=rank, world_size=world)


def _history_worker(rank, world, port_no, out, bc, rel_tol):
    _init(rank, world, port_no)
    try:
        op, B = _problem(bc)
        plan = shard.BlockPlan(m=26, n=26, world=world, rank=rank, h=shard.halo_rows(op))
        Bl = torch.from_numpy(B[plan.g0:plan.g0 + plan.rows].copy())
        X, hist = shard.solve_row_blocks(DenseBlockBackend(op, plan), plan, Bl, 1.3, 0.05, 25, project=True,
                                         record_history=True, rel_tol=rel_tol)
        parts = [torch.zeros((r, 26), dtype=torch.float64) for _, r in plan.parts]
        dist.all_gather(parts, X)
        if rank == 0:
            out.put((torch.cat(parts).numpy(), hist))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("bc", ["zero", "reflective"])
def test_row_block_history_norms_are_all_reduced(bc):
    """record_history on 2 ranks: the per-iteration norms (solvers.py:178-179) and objective
    (solvers.py:133-141, 187) are the global ones -- equal to the reference loop's on one image."""
    x, hist = _run_world2(_history_worker, bc, 0.0)
    op, B = _problem(bc)
    pop = port.PortOperator(op)
    xp = np.zeros_like(B)
    _, beta = kb.momentum_table(25)
    y = xp.copy()
    for k in range(1, 26):
        xk = np.maximum((1.3 * y - port.kron_apply_adjoint(pop, port.kron_apply(pop, y) - B)) / (1.3 + 0.05**2), 0)
        h = hist[k - 1]
        assert h["k"] == k
        assert h["step2"] == pytest.approx(float(np.sum((xk - xp) ** 2)), rel=1e-10, abs=1e-300)
        assert h["base2"] == pytest.approx(float(np.sum(xp ** 2)), rel=1e-10, abs=1e-300)
        assert h["x2"] == pytest.approx(float(np.sum(xk ** 2)), rel=1e-10)
        r = port.kron_apply(pop, xk) - B
        assert h["objective"] == pytest.approx(0.5 * float(np.sum(r * r)) + 0.5 * 0.05**2 * float(np.sum(xk * xk)),
                                               rel=1e-10)
        y = xk + beta[k - 1] * (xk - xp)
        xp = xk
    np.testing.assert_allclose(x, xp, rtol=0, atol=1e-12 * np.abs(xp).max())


def test_row_block_rel_tol_stops_on_global_norms():
    x, hist = _run_world2(_history_worker, "zero", 5e-2)
    op, B = _problem("zero")
    # the reference's stopping rule on the global norms, replayed on one image
    want, _ = port.sfista(op, B, 1.3, 0.05, len(hist), project=True)
    assert len(hist) < 25
    s = [np.sqrt(h["step2"]) < 5e-2 * np.sqrt(h["base2"]) for h in hist]
    assert s[-1] and not any(s[:-1])
    np.testing.assert_allclose(x, want, rtol=0, atol=1e-12 * np.abs(want).max())


def _power_worker(rank, world, port_no, out, bc):
    _init(rank, world, port_no)
    try:
        op, _ = _problem(bc)
        plan = shard.BlockPlan(m=26, n=26, world=world, rank=rank, h=shard.halo_rows(op))
        v0 = port.lipschitz_start(3, (26, 26))
        L = shard.power_iter_row_blocks(DenseBlockBackend(op, plan), plan,
                                        torch.from_numpy(v0[plan.g0:plan.g0 + plan.rows].copy()), 50)
        if rank == 0:
            out.put(L)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("bc", ["zero", "reflective"])
def test_sharded_power_iteration_matches_reference_loop(bc):
    """estimate_lipschitz (solvers.py:104-130) with <v, w> and ||w||^2 all-reduced over 2 ranks."""
    L = _run_world2(_power_worker, bc)
    op, _ = _problem(bc)
    pop = port.PortOperator(op)
    want = port.estimate_lipschitz(lambda v: port.kron_apply(pop, v), lambda v: port.kron_apply_adjoint(pop, v),
                                   (26, 26), 50, 3)
    assert L == pytest.approx(want, rel=1e-12)


def _batch_worker(rank, world, port_no, out):
    _init(rank, world, port_no)
    try:
        ops, Bs, Ls = _batch_problem()

        def cpu_solver(ops_s, B_s, L_s, lam, iters, opts):
            return np.stack([port.sfista(o, b, l, lam, iters, project=True)[0] for o, b, l in zip(ops_s, B_s, L_s)]), 0.0

        start, x, _ = shard.solve_batch_shard(ops, Bs, Ls, 0.02, 15, rank, world, solver=cpu_solver)
        got = [None] * world
        dist.all_gather_object(got, (start, x))
        if rank == 0:
            out.put(got)
    finally:
        dist.destroy_process_group()


def _batch_problem():
    rng = np.random.default_rng(5)
    ops, Bs = [], []
    for i in range(5):
        op = kb.decompose(random_psf(rng, 5), kb.BoundaryCondition("zero"), s=2, shape=(20, 20))
        ops.append(op)
        Bs.append(rng.random((20, 20)))
    return ops, np.stack(Bs), np.linspace(1.1, 1.3, 5)


def test_batch_shard_world2_partitions_without_communication():
    """cfg3-style batch sharding on 2 ranks: each rank solves its contiguous slice of independent
    images (3 + 2 of 5); the gathered slices equal the per-image solves."""
    got = _run_world2(_batch_worker)
    ops, Bs, Ls = _batch_problem()
    assert [g[0] for g in got] == [0, 3] and [len(g[1]) for g in got] == [3, 2]
    x = np.concatenate([g[1] for g in got])
    for i in range(5):
        want, _ = port.sfista(ops[i], Bs[i], Ls[i], 0.02, 15, project=True)
        np.testing.assert_allclose(x[i], want, rtol=0, atol=1e-13)


def test_prefer_swap_rule():
    """The bench's sharded axis swap follows kb_op_create's twin rule: large fp32 images whose
    axis-1 band is >= 8 wider than the axis-0 band."""
    from paper_1901_00913_b200 import workloads as W

    cfg5 = W.CONFIGS["cfg5"]
    op = kb.decompose(W.make_psf(cfg5), kb.BoundaryCondition("reflective"), s=10, shape=(16384, 16384))
    assert shard.prefer_swap(op, "float32") and not shard.prefer_swap(op, "float64")
    sw = shard.swapped(op)
    assert shard.halo_rows(sw) >= shard.halo_rows(op) + 8 and not shard.prefer_swap(sw, "float32")
    assert sw.terms[0].H is op.terms[0].K and sw.shape == (16384, 16384)
