"""Multi-GPU execution of the sFISTA hot path. One process per GPU.

* Batch sharding (BASELINE cfg3): independent images are split across ranks; every rank runs the
  batched native loop on its slice. No collective touches the data path.
* Row-block sharding (cfg4, cfg5): a single image is split into contiguous row blocks. The axis-0
  factor H_i needs +-h neighbour rows (h = half band width), so before each forward and each
  adjoint application the block exchanges h halo rows with its neighbours (one grouped
  send/recv per neighbour over NCCL / NVLink; gloo for the CPU tests). Axis 1 is local. Only the
  first and last ranks see the global domain edges, where the kernels apply the zero / reflective
  rule (global row indices g0 / m_global are passed down, structured.py:111-123).

The local arithmetic goes through a backend with two calls — residual (R = A Y - B on the block)
and update (adjoint + FISTA update on the block). ``DeviceBlockBackend`` runs the C-ABI kernels
(kb_block_residual / kb_block_update); tests substitute a dense CPU backend to check the partition
and halo plumbing with world_size 2 on gloo.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from .errors import ArgumentError, NumericError


def row_partition(m: int, world: int) -> list[tuple[int, int]]:
    """Contiguous balanced row blocks: [(g0, rows)] per rank."""
    if world < 1 or m < world:
        raise ArgumentError(f"cannot split {m} rows over {world} ranks")
    base, extra = divmod(m, world)
    out, g0 = [], 0
    for r in range(world):
        rows = base + (1 if r < extra else 0)
        out.append((g0, rows))
        g0 += rows
    return out


def halo_rows(op) -> int:
    """Axis-0 halo: the largest |offset| of any H_i stencil band."""
    from .structured import factor_band

    h = 0
    for t in op.terms:
        dlo, taps = factor_band(t.H)
        h = max(h, abs(dlo), abs(dlo + taps.size - 1))
    return h


def batch_partition(batch: int, world: int) -> list[tuple[int, int]]:
    """Contiguous balanced image ranges: [(start, count)] per rank (counts may be 0)."""
    base, extra = divmod(batch, world)
    out, s = [], 0
    for r in range(world):
        c = base + (1 if r < extra else 0)
        out.append((s, c))
        s += c
    return out


@dataclass
class BlockPlan:
    m: int
    n: int
    world: int
    rank: int
    h: int  # halo rows (axis-0 half band width)

    def __post_init__(self):
        self.parts = row_partition(self.m, self.world)
        self.g0, self.rows = self.parts[self.rank]
        if self.world > 1 and min(r for _, r in self.parts) < self.h:
            raise ArgumentError(f"row blocks of {min(r for _, r in self.parts)} rows are thinner "
                                f"than the halo ({self.h}); use fewer ranks")
        self.prev = self.rank - 1 if self.rank > 0 else None
        self.next = self.rank + 1 if self.rank < self.world - 1 else None
        self.hlo = self.h if self.prev is not None else 0
        self.hhi = self.h if self.next is not None else 0


def exchange_halos(buf, plan: BlockPlan, group=None):
    """buf: [h + rows + h, n] tensor (interior at rows h .. h+rows-1). Fills the halo rows from
    the neighbours: my first h interior rows go to prev (its bottom halo), my last h to next."""
    import torch.distributed as dist

    h, rows = plan.h, plan.rows
    if plan.world == 1 or h == 0:
        return
    ops = []
    if plan.prev is not None:
        ops.append(dist.P2POp(dist.isend, buf[h : 2 * h].contiguous(), plan.prev, group))
        top = buf[0:h]
        ops.append(dist.P2POp(dist.irecv, top, plan.prev, group))
    if plan.next is not None:
        ops.append(dist.P2POp(dist.isend, buf[rows : rows + h].contiguous(), plan.next, group))
        bot = buf[h + rows : 2 * h + rows]
        ops.append(dist.P2POp(dist.irecv, bot, plan.next, group))
    for req in dist.batch_isend_irecv(ops):
        req.wait()


class DeviceBlockBackend:
    """Row-block kernels of libkb_b200.so for one rank (operator uploaded with m = rows)."""

    def __init__(self, op, plan: BlockPlan, dtype: str = "float32"):
        from . import device as D

        self.plan = plan
        self.dev = D.DeviceOperator([_LocalShape(op, plan.rows)], dtype)
        self.D = D
        if plan.world > 1 and self.dev.half_widths[0] > plan.h:
            raise ArgumentError("halo narrower than the axis-0 band")

    def residual(self, Yh, B, R):
        p, D = self.plan, self.D
        y0 = Yh[p.h:]
        r0 = R[p.h:]
        rc = D.load_library().kb_block_residual(self.dev._handle, D._ptr(y0), D._ptr(B), D._ptr(r0),
                                                D._ptr(self.dev.work), p.g0, p.m, p.hlo, p.hhi,
                                                D._stream_handle())
        D._check(rc, "kb_block_residual")

    def update(self, Rh, X, Yh, beta, k, L, lam, project, flag):
        p, D = self.plan, self.D
        rc = D.load_library().kb_block_update(self.dev._handle, D._ptr(Rh[p.h:]), D._ptr(X),
                                              D._ptr(Yh[p.h:]), D._ptr(self.dev.work), p.g0, p.m,
                                              p.hlo, p.hhi, float(beta), int(k), float(L), float(lam),
                                              int(bool(project)), D._ptr(flag), D._stream_handle())
        D._check(rc, "kb_block_update")


class _LocalShape:
    """View of a KronOperator whose axis-0 factor order is the local block height (the device
    tables hold bands only; the global row geometry is passed per call)."""

    def __init__(self, op, rows):
        self.shape = (rows, op.shape[1])
        self.terms = tuple(_LocalTerm(t, rows) for t in op.terms)
        self.bc = op.bc


class _LocalTerm:
    def __init__(self, t, rows):
        self.sigma, self.K = t.sigma, t.K
        self.H = _Resized(t.H, rows)


class _Resized:
    """Factor with the same stencil band (read from c and j by factor_band) but declared order
    `rows`: the device operator of a row block."""

    def __init__(self, f, rows):
        self.kind, self.c, self.j, self.n = f.kind, f.c, f.j, rows


def solve_row_blocks(backend, plan: BlockPlan, B_local, L: float, lam: float, iters: int,
                     project: bool = True, group=None, X0_local=None, sync=None):
    """sFISTA on a row-sharded image (solvers.py:168-174 per iteration, two halo exchanges).

    B_local: [rows, n] tensor of this rank's data rows. Returns x_iters on the rank's rows.
    `sync` (optional) is called after each exchange-compute step (device timing hooks)."""
    import torch

    from .device import INT_MAX
    from .solvers import momentum_table

    h, rows, n = plan.h, plan.rows, plan.n
    _, beta = momentum_table(int(iters))
    Yh = torch.zeros((rows + 2 * h, n), dtype=B_local.dtype, device=B_local.device)
    Rh = torch.zeros_like(Yh)
    X = torch.zeros((rows, n), dtype=B_local.dtype, device=B_local.device)
    if X0_local is not None:
        X.copy_(X0_local)
        Yh[h:h + rows].copy_(X0_local)
    flag = torch.full((1,), INT_MAX, dtype=torch.int32, device=B_local.device)
    for k in range(1, int(iters) + 1):
        exchange_halos(Yh, plan, group)
        backend.residual(Yh, B_local, Rh)
        exchange_halos(Rh, plan, group)
        backend.update(Rh, X, Yh, beta[k - 1], k, L, lam, project, flag)
        if sync is not None:
            sync(k)
    bad = int(flag.item())
    if bad <= iters:
        raise NumericError(f"non-finite iterate at iteration {bad}")
    return X


def solve_batch_shard(ops, B, L, lam: float, iters: int, rank: int, world: int, options=None):
    """Batch sharding: this rank solves images [start, start+count) of the batch with no
    communication. Returns (start, x_slice, solve_ms)."""
    from .device import DeviceOperator
    from .solvers import sfista_batch

    start, count = batch_partition(len(ops), world)[rank]
    if count == 0:
        return start, None, 0.0
    dev = DeviceOperator(list(ops[start:start + count]), options.dtype if options else "float32")
    x, ms = sfista_batch(dev, B[start:start + count], np.asarray(L)[start:start + count], lam, iters,
                         options=options)
    return start, x, ms
