"""Multi-GPU execution of the sFISTA hot path. One process per GPU.

* Batch sharding (BASELINE cfg3): independent images are split across ranks; every rank runs the
  batched native loop on its slice. No collective touches the data path.
* Row-block sharding (cfg4, cfg5): a single image is split into contiguous row blocks. The axis-0
  factor H_i needs +-h neighbour rows (h = half band width), so before each forward and each
  adjoint application the block exchanges h halo rows with its neighbours (one grouped
  send/recv per neighbour over NCCL / NVLink; gloo for the CPU tests). Axis 1 is local. Only the
  first and last ranks see the global domain edges, where the kernels apply the zero / reflective
  rule (global row indices g0 / m_global are passed down, structured.py:111-123).
* Overlap: when the halo is a sizeable share of the block (cfg4 at 8 ranks: 127 of 512 rows),
  each half-iteration computes the interior rows [h, rows-h) -- which need no halo -- while the
  exchange is in flight, then the two h-row edge strips once it has landed. For thin halos (cfg5:
  14 of 2048 rows) the extra launches cost more than the ~10 us exchange, and the block runs whole.
* Scalars: history / rel_tol norms (solvers.py:178-192) and the power iteration's <v, w>, ||w||^2
  (solvers.py:124-125) are partial sums per block, all-reduced (fp64 sum) across the ranks.

The local arithmetic goes through a backend -- residual (R = A Y - B on rows [r0, r1) of the
block), update (adjoint + FISTA update on rows [r0, r1)), apply and inner2 (power iteration).
``DeviceBlockBackend`` runs the C-ABI kernels (kb_block_residual / kb_block_update /
kb_apply_block / kb_inner2); the CPU tests substitute a dense backend to check the partition,
halo plumbing and collectives with world_size 2 on gloo.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import ArgumentError, NumericError

OVERLAP_MIN_HALO_FRACTION = 0.05  # overlap the exchange when h / rows is at least this


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


def halo_rows(op, rel_tol: float | None = None) -> int:
    """Axis-0 halo: the largest |offset| of any H_i stencil band, with the band trimmed exactly
    as the device operator trims it (device.BAND_REL_TOL: reflective generators carry ~1e-16
    leakage over half the axis, which would otherwise make the halo the whole image)."""
    from .device import BAND_REL_TOL
    from .structured import factor_band

    tol = BAND_REL_TOL if rel_tol is None else rel_tol
    h = 0
    for t in op.terms:
        dlo, taps = factor_band(t.H, tol)
        h = max(h, abs(dlo), abs(dlo + taps.size - 1))
    return h


def swapped(op):
    """The operator of the transposed image, Y^T = sum_i K_i X^T H_i^T (H and K swapped)."""
    from .kron import KronOperator, KronTerm

    return KronOperator(terms=tuple(KronTerm(sigma=t.sigma, H=t.K, K=t.H) for t in op.terms),
                        shape=(op.shape[1], op.shape[0]), bc=op.bc, sigma=op.sigma, s=op.s, rank=op.rank,
                        eps=op.eps)


def prefer_swap(op, dtype: str) -> bool:
    """kb_op_create's axis-swap rule (large fp32 images whose axis-1 band is >= 8 wider than the
    axis-0 band run the wider band in pass A): the sharded solve then splits the TRANSPOSED image
    into row blocks, so N > 1 runs the same kernels as the single-GPU fast path."""
    import os

    env = os.environ.get("KB_AXIS_SWAP")
    if env is not None:
        return env == "1"
    if dtype != "float32" or op.shape[0] * op.shape[1] < 4096 * 4096:
        return False
    return halo_rows(swapped(op)) >= halo_rows(op) + 8


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

    def sub(self, r0: int, r1: int):
        """Geometry of local rows [r0, r1): (global first row, halo rows readable above and
        below -- local rows of the block plus the exchanged halo)."""
        return (self.g0 + r0, min(self.h, r0 + self.hlo), min(self.h, self.rows - r1 + self.hhi))

    def overlap_ranges(self):
        """[(r0, r1)] interior first, then the edge strips, or None when not worth it."""
        h, rows = self.h, self.rows
        if self.world == 1 or h == 0 or rows < 3 * h or h < OVERLAP_MIN_HALO_FRACTION * rows:
            return None
        return [(h, rows - h)], [(0, h), (rows - h, rows)]


def exchange_halos(buf, plan: BlockPlan, group=None, async_op: bool = False):
    """buf: [h + rows + h, n] tensor (interior at rows h .. h+rows-1). Fills the halo rows from
    the neighbours: my first h interior rows go to prev (its bottom halo), my last h to next.
    async_op=True returns the pending works (NCCL runs them on its own stream; .wait() orders
    the caller's stream after them) so computation can proceed meanwhile."""
    import torch.distributed as dist

    h, rows = plan.h, plan.rows
    if plan.world == 1 or h == 0:
        return []
    ops = []
    if plan.prev is not None:
        ops.append(dist.P2POp(dist.isend, buf[h: 2 * h], plan.prev, group))
        ops.append(dist.P2POp(dist.irecv, buf[0:h], plan.prev, group))
    if plan.next is not None:
        ops.append(dist.P2POp(dist.isend, buf[rows: rows + h], plan.next, group))
        ops.append(dist.P2POp(dist.irecv, buf[h + rows: 2 * h + rows], plan.next, group))
    works = dist.batch_isend_irecv(ops)
    if async_op:
        return works
    for req in works:
        req.wait()
    return []


def all_reduce_sum(t, plan: BlockPlan, group=None):
    """fp64 sum of per-block partials across the ranks (in place)."""
    if plan.world > 1:
        import torch.distributed as dist

        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return t


class DeviceBlockBackend:
    """Row-block kernels of libkb_b200.so for one rank. One device operator per row-range height
    (the device tables hold bands only; global row geometry is passed per call)."""

    def __init__(self, op, plan: BlockPlan, dtype: str = "float32"):
        from . import device as D

        self.op, self.plan, self.dtype, self.D = op, plan, dtype, D
        self._devs = {}
        dev = self.dev = self._dev(plan.rows)
        if plan.world > 1 and dev.half_widths[0] > plan.h:
            raise ArgumentError("halo narrower than the axis-0 band")
        self._work2 = None

    def _dev(self, height):
        dev = self._devs.get(height)
        if dev is None:
            dev = self._devs[height] = self.D.DeviceOperator([_LocalShape(self.op, height)], self.dtype)
        return dev

    def residual(self, Yh, B, R, r0=0, r1=None):
        p, D = self.plan, self.D
        r1 = p.rows if r1 is None else r1
        g0, hlo, hhi = p.sub(r0, r1)
        dev = self._dev(r1 - r0)
        rc = D.load_library().kb_block_residual(dev._handle, D._ptr(Yh[p.h + r0:]), D._ptr(B[r0:]),
                                                D._ptr(R[p.h + r0:]), D._ptr(dev.work), g0, p.m, hlo, hhi,
                                                D._stream_handle())
        D._check(rc, "kb_block_residual")

    def update(self, Rh, X, Yh, beta, k, L, lam, project, flag, r0=0, r1=None, norms=None):
        p, D = self.plan, self.D
        r1 = p.rows if r1 is None else r1
        g0, hlo, hhi = p.sub(r0, r1)
        dev = self._dev(r1 - r0)
        rc = D.load_library().kb_block_update(dev._handle, D._ptr(Rh[p.h + r0:]), D._ptr(X[r0:]),
                                              D._ptr(Yh[p.h + r0:]), D._ptr(dev.work), g0, p.m, hlo, hhi,
                                              float(beta), int(k), float(L), float(lam), int(bool(project)),
                                              D._ptr(flag), D._ptr(norms) if norms is not None else None,
                                              D._stream_handle())
        D._check(rc, "kb_block_update")

    def apply(self, Xh, out, adjoint=False):
        """out[rows] = (A or A^T) X on the block; Xh carries the exchanged halo rows."""
        p, D = self.plan, self.D
        g0, hlo, hhi = p.sub(0, p.rows)
        rc = D.load_library().kb_apply_block(self.dev._handle, int(bool(adjoint)), D._ptr(Xh[p.h:]),
                                             D._ptr(out), D._ptr(self.dev.work), g0, p.m, hlo, hhi,
                                             D._stream_handle())
        D._check(rc, "kb_apply_block")

    def resid2(self, AX, B, out2):
        """out2[0] (device double) = ||AX - B||^2 over this block (kb_resid_norms)."""
        import torch

        D = self.D
        if self._work2 is None:
            self._work2 = torch.empty(D.KB_RESID_NORMS_WORK // 8, dtype=torch.float64, device=AX.device)
        rc = D.load_library().kb_resid_norms(D._code(self.dtype), D._ptr(AX), D._ptr(B), None, None, int(AX.numel()),
                                             D._ptr(out2), D._ptr(self._work2), D._stream_handle())
        D._check(rc, "kb_resid_norms")

    def inner2(self, a, b, out2):
        """out2 (device double[2]) = <a, b>, ||b||^2 over this block (kb_inner2)."""
        import torch

        D = self.D
        if self._work2 is None:
            self._work2 = torch.empty(D.KB_RESID_NORMS_WORK // 8, dtype=torch.float64, device=a.device)
        rc = D.load_library().kb_inner2(D._code(self.dtype), D._ptr(a), D._ptr(b), int(b.numel()), D._ptr(out2),
                                        D._ptr(self._work2), D._stream_handle())
        D._check(rc, "kb_inner2")


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


def _phase(backend, plan, buf, group, compute, overlap):
    """Exchange buf's halo rows and run compute(r0, r1) over the block: with overlap, the
    interior rows while the exchange is in flight, then the edge strips."""
    ranges = plan.overlap_ranges() if overlap else None
    if ranges is None:
        exchange_halos(buf, plan, group)
        compute(0, plan.rows)
        return
    inner, edges = ranges
    works = exchange_halos(buf, plan, group, async_op=True)
    for r0, r1 in inner:
        compute(r0, r1)
    for req in works:
        req.wait()
    for r0, r1 in edges:
        compute(r0, r1)


def solve_row_blocks(backend, plan: BlockPlan, B_local, L: float, lam: float, iters: int,
                     project: bool = True, group=None, X0_local=None, sync=None, rel_tol: float = 0.0,
                     record_history: bool = False, overlap: bool = True):
    """sFISTA on a row-sharded image (solvers.py:168-198 per iteration, two halo exchanges).

    B_local: [rows, n] tensor of this rank's data rows. Returns x on the rank's rows, or
    (x, history) with record_history / rel_tol, history[k-1] = dict of the all-reduced
    ||x_k - x_{k-1}||^2, ||x_{k-1}||^2, ||x_k||^2 and (record_history) ||A x_k - b||^2 with the
    objective 1/2 ||A x_k - b||^2 + lam^2/2 ||x_k||^2 (solvers.py:133-141, 178-192); rel_tol stops
    as solvers.py:197-198 on the GLOBAL norms. `sync` (optional) is called after each iteration."""
    import torch

    from .device import INT_MAX
    from .solvers import momentum_table

    h, rows, n = plan.h, plan.rows, plan.n
    _, beta = momentum_table(int(iters))
    dev = B_local.device
    Yh = torch.zeros((rows + 2 * h, n), dtype=B_local.dtype, device=dev)
    Rh = torch.zeros_like(Yh)
    X = torch.zeros((rows, n), dtype=B_local.dtype, device=dev)
    if X0_local is not None:
        X.copy_(X0_local)
        Yh[h:h + rows].copy_(X0_local)
    flag = torch.full((1,), INT_MAX, dtype=torch.int32, device=dev)
    want_norms = record_history or rel_tol > 0
    norms = torch.zeros(8, dtype=torch.float64, device=dev) if want_norms else None
    part = torch.zeros(8, dtype=torch.float64, device=dev) if want_norms else None
    history = []
    Xh = torch.zeros_like(Yh) if record_history else None
    AX = torch.zeros((rows, n), dtype=B_local.dtype, device=dev) if record_history else None
    for k in range(1, int(iters) + 1):
        _phase(backend, plan, Yh, group, lambda r0, r1: backend.residual(Yh, B_local, Rh, r0, r1), overlap)
        if want_norms:
            norms.zero_()

        def upd(r0, r1):
            if not want_norms:
                backend.update(Rh, X, Yh, beta[k - 1], k, L, lam, project, flag, r0, r1)
                return
            backend.update(Rh, X, Yh, beta[k - 1], k, L, lam, project, flag, r0, r1, norms=part)
            norms[:3] += part[:3]

        _phase(backend, plan, Rh, group, upd, overlap)
        if want_norms:
            if record_history:  # ||A x_k - b||^2 on the block: x halo exchange + block forward
                Xh[h:h + rows].copy_(X)
                exchange_halos(Xh, plan, group)
                backend.apply(Xh, AX)
                backend.resid2(AX, B_local, part)
                norms[3] = part[0]
            all_reduce_sum(norms, plan, group)
            step2, base2, x2, r2 = (float(v) for v in norms[:4].cpu())
            rec = {"k": k, "step2": step2, "base2": base2, "x2": x2}
            if record_history:
                rec["resid2"] = r2
                rec["objective"] = 0.5 * r2 + 0.5 * lam ** 2 * x2
            history.append(rec)
            if int(flag.item()) <= k:
                raise NumericError(f"non-finite iterate at iteration {k}")
        if sync is not None:
            sync(k)
        if rel_tol > 0:
            step, base = np.sqrt(history[-1]["step2"]), np.sqrt(history[-1]["base2"])
            if step < rel_tol * (base if base > 0 else 1.0):
                break
    bad = int(flag.item())
    if bad <= iters:
        raise NumericError(f"non-finite iterate at iteration {bad}")
    return (X, history) if want_norms else X


def power_iter_row_blocks(backend, plan: BlockPlan, v_local, iters: int = 50, group=None) -> float:
    """estimate_lipschitz (solvers.py:104-130) on a row-sharded operand: per step the halo of v
    is exchanged, u = A v and w = A^T u run on the block (u's halo exchanged in between), and the
    block partials <v, w>, ||w||^2 are all-reduced before v = w / ||w||. v_local: this rank's
    rows of the normalised start vector (the same global Philox draw on every rank)."""
    import torch
    import warnings

    from .solvers import LIPSCHITZ_SAFETY

    h, rows, n = plan.h, plan.rows, plan.n
    dev = v_local.device
    Vh = torch.zeros((rows + 2 * h, n), dtype=v_local.dtype, device=dev)
    Uh = torch.zeros_like(Vh)
    W = torch.zeros((rows, n), dtype=v_local.dtype, device=dev)
    Vh[h:h + rows].copy_(v_local)
    red = torch.zeros(2, dtype=torch.float64, device=dev)
    rho = 0.0
    for _ in range(int(iters)):
        exchange_halos(Vh, plan, group)
        backend.apply(Vh, Uh[h:h + rows])
        exchange_halos(Uh, plan, group)
        backend.apply(Uh, W, adjoint=True)
        backend.inner2(Vh[h:h + rows], W, red)
        all_reduce_sum(red, plan, group)
        rho, nw2 = (float(x) for x in red.cpu())
        if nw2 == 0 or rho <= 0:
            warnings.warn("operator is numerically zero; Lipschitz floor returned")
            return float(np.finfo(float).eps)
        Vh[h:h + rows].copy_(W / np.sqrt(nw2))
    return LIPSCHITZ_SAFETY * rho


def solve_batch_shard(ops, B, L, lam: float, iters: int, rank: int, world: int, options=None, solver=None):
    """Batch sharding: this rank solves images [start, start+count) of the batch with no
    communication. Returns (start, x_slice, solve_ms). `solver(ops_slice, B_slice, L_slice, lam,
    iters, options) -> (x, ms)` defaults to the batched device solve (sfista_batch)."""
    start, count = batch_partition(len(ops), world)[rank]
    if count == 0:
        return start, None, 0.0
    sl = slice(start, start + count)
    if solver is None:
        from .device import DeviceOperator
        from .solvers import sfista_batch

        def solver(ops_s, B_s, L_s, lam_, iters_, opts):
            dev = DeviceOperator(list(ops_s), opts.dtype if opts else "float32")
            return sfista_batch(dev, B_s, L_s, lam_, iters_, options=opts)
    x, ms = solver(list(ops[sl]), B[sl], np.asarray(L)[sl], lam, iters, options)
    return start, x, ms
