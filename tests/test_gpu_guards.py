"""Guard bands around every buffer a kernel family touches (the write checks of memcheck, which
this GPU pool does not allow): operands, outputs and the operator workspace are views into larger
allocations whose margins hold a canary; after apply / adjoint / sFISTA (fast, history and
row-block paths) / power iteration / blur on each kernel family the margins must be untouched.
"""

import numpy as np
import pytest

from conftest import cuda_ok, random_psf

pytestmark = pytest.mark.gpu

if not cuda_ok():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import torch  # noqa: E402

import paper_1901_00913_b200 as kb  # noqa: E402
from paper_1901_00913_b200.device import INT_MAX, DeviceOperator  # noqa: E402

GUARD = 4096  # elements (>= 16 KB) on each side
CANARY = -12345.678


class Guarded:
    """A plane view inside a canary-filled allocation."""

    def __init__(self, shape, dtype, fill=None):
        n = int(np.prod(shape))
        self.buf = torch.full((GUARD + n + GUARD,), CANARY, dtype=dtype, device="cuda")
        self.t = self.buf[GUARD:GUARD + n].view(*shape)
        if fill is not None:
            self.t.copy_(fill)

    def check(self, what):
        torch.cuda.synchronize()
        lo, hi = self.buf[:GUARD], self.buf[-GUARD:]
        assert bool((lo == CANARY).all()) and bool((hi == CANARY).all()), f"{what}: write outside the buffer"


def guard_workspace(dev):
    """Move the operator's workspace into a guarded allocation (byte canary 0xA5)."""
    nbytes = dev.work.numel()
    buf = torch.full((GUARD * 8 + nbytes + GUARD * 8,), 0xA5, dtype=torch.uint8, device="cuda")
    dev.work = buf[GUARD * 8:GUARD * 8 + nbytes]

    def check(what):
        torch.cuda.synchronize()
        assert bool((buf[:GUARD * 8] == 0xA5).all()) and bool((buf[-GUARD * 8:] == 0xA5).all()), \
            f"{what}: write outside the workspace"
    return check


CASES = [  # (name, m, n, batch, psf size, bc, dtype)
    ("dmma", 192, 160, 1, 9, "reflective", "float64"),
    ("dmma_zero", 192, 160, 1, 9, "zero", "float64"),
    ("generic_odd", 45, 37, 1, 7, "reflective", "float64"),
    ("mma_tf32", 192, 160, 1, 9, "reflective", "float32"),
    ("tcgen05", 1024, 1024, 1, 129, "zero", "float32"),
    ("tcgen05_refl", 1024, 1024, 1, 129, "reflective", "float32"),
    ("batched", 96, 96, 3, 7, "zero", "float32"),
    ("batched64", 96, 96, 3, 7, "reflective", "float64"),
]


@pytest.mark.parametrize("name,m,n,batch,w,bc,dtype", CASES)
def test_no_writes_outside_buffers(name, m, n, batch, w, bc, dtype):
    rng = np.random.default_rng(len(name) * 31 + m)
    if m != n:
        m = n = max(m, n)  # decompose wants square images
    ops = [kb.decompose(random_psf(rng, w), kb.BoundaryCondition(bc), s=3, shape=(m, n)) for _ in range(batch)]
    dev = DeviceOperator(ops, dtype)
    check_ws = guard_workspace(dev)
    shape = (batch, m, n) if batch > 1 else (m, n)
    td = dev.tdtype
    X = Guarded(shape, td, torch.from_numpy(rng.random(shape)).to(td))
    Y = Guarded(shape, td)
    for adjoint in (False, True):
        dev.apply(X.t, out=Y.t, adjoint=adjoint)
        X.check(f"{name} apply input")
        Y.check(f"{name} apply output (adjoint={adjoint})")
        check_ws(f"{name} apply")
    B = Guarded(shape, td, torch.from_numpy(rng.random(shape)).to(td))
    Xs, Ys = Guarded(shape, td, 0.0), Guarded(shape, td, 0.0)
    flag = torch.full((1,), INT_MAX, dtype=torch.int32, device="cuda")
    _, beta = kb.momentum_table(4)
    norms = torch.zeros((4, 4, batch), dtype=torch.float64, device="cuda")
    for use_norms in (False, True):
        dev.sfista_run(B.t, Xs.t, Ys.t, beta, 0, 4, np.full(batch, 1.3), 0.03, True, flag,
                       norms=norms if use_norms else None)
        for g, what in ((B, "data"), (Xs, "x"), (Ys, "y")):
            g.check(f"{name} sfista {what} (norms={use_norms})")
        check_ws(f"{name} sfista")
    V = Guarded(shape, td, torch.from_numpy(rng.standard_normal(shape) / np.sqrt(np.prod(shape))).to(td))
    dev.power_iter(V.t, 3)
    V.check(f"{name} power iteration")
    check_ws(f"{name} power iteration")


@pytest.mark.parametrize("bc", ["zero", "reflective"])
def test_blur_no_writes_outside(bc):
    from paper_1901_00913_b200 import device as D

    rng = np.random.default_rng(3)
    psf = random_psf(rng, 9)
    X = Guarded((70, 66), torch.float64, torch.from_numpy(rng.random((70, 66))))
    Y = Guarded((70, 66), torch.float64)
    P = torch.from_numpy(np.ascontiguousarray(psf.values)).cuda()
    rc = D.load_library().kb_blur_direct(D._ptr(P), 0, 9, 9, psf.center[0], psf.center[1], D._ptr(X.t),
                                         D._ptr(Y.t), 70, 66, 1, 1 if bc == "reflective" else 0, D._stream_handle())
    D._check(rc, "kb_blur_direct")
    X.check("blur input")
    Y.check("blur output")
