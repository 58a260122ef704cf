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
    """R = A Y - B and the projected FISTA update on rows [g0, g0+rows), from dense factors."""

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

    def residual(self, Yh, B, R):
        p = self.plan
        rows, cols = slice(p.g0, p.g0 + p.rows), self._cols()
        Y = self._halo(Yh)
        acc = sum(Ha[rows, cols] @ Y @ Kb.T for Ha, Kb in zip(self.Ha, self.Kb))
        R[p.h:p.h + p.rows] = torch.from_numpy(acc - B.numpy())

    def update(self, Rh, X, Yh, beta, k, L, lam, project, flag):
        p = self.plan
        rows, cols = slice(p.g0, p.g0 + p.rows), self._cols()
        Rm = self._halo(Rh)
        G = sum(Ha.T[rows, cols] @ Rm @ Kb for Ha, Kb in zip(self.Ha, self.Kb))
        y = Yh[p.h:p.h + p.rows].numpy()
        xp = X.numpy().copy()
        x = (L * y - G) / (L + lam**2)
        if project:
            x = np.maximum(x, 0.0)
        X.copy_(torch.from_numpy(x))
        Yh[p.h:p.h + p.rows] = torch.from_numpy(x + beta * (x - xp))


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
