import sys, numpy as np, torch
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import paper_1901_00913_b200 as kb
from paper_1901_00913_b200 import shard, device as D
from oracle import kronblur_port as port
from conftest import random_psf
rng = np.random.default_rng(20240817)
for bc in ("zero", "reflective"):
    psf = random_psf(rng, 9)
    op = kb.decompose(psf, kb.BoundaryCondition(bc), s=3, shape=(90, 90))
    h = shard.halo_rows(op)
    X = rng.standard_normal((90, 90))
    full = port.kron_apply(port.PortOperator(op), X); fullT = port.kron_apply_adjoint(port.PortOperator(op), X)
    for g0, rows in ((0, 30), (30, 30), (60, 30)):
        hlo = h if g0 > 0 else 0; hhi = h if g0 + rows < 90 else 0
        dev = D.DeviceOperator([shard._LocalShape(op, rows)], "float64")
        buf = np.zeros((rows + 2 * h, 90)); buf[h - hlo:h + rows + hhi] = X[g0 - hlo:g0 + rows + hhi]
        Xh = torch.from_numpy(buf).cuda()
        out = torch.empty((rows, 90), dtype=torch.float64, device="cuda")
        for adj, want in ((0, full), (1, fullT)):
            rc = D.load_library().kb_apply_block(dev._handle, adj, D._ptr(Xh[h:]), D._ptr(out), D._ptr(dev.work), g0, 90, hlo, hhi, D._stream_handle())
            D._check(rc, "x")
            err = np.abs(out.cpu().numpy() - want[g0:g0 + rows]).max()
            print(bc, "h", h, "block", g0, "adj", adj, "err %.2e" % err)
# full-image forward for comparison, plus the two passes separately via shapes
for m in (90, 30, 32, 34, 64):
    psf = random_psf(np.random.default_rng(1), 9)
    op = kb.decompose(psf, kb.BoundaryCondition("reflective"), s=3, shape=(m, m))
    X = np.random.default_rng(2).standard_normal((m, m))
    got = kb.kron_apply(op, X)
    want = port.kron_apply(port.PortOperator(op), X)
    print("full", m, "err %.2e" % np.abs(got - want).max())
