"""Per-case debug run of tests/fused_cases.py's operator cases (KB_FUSED=1 KB_FUSED_TRACE=1)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np, torch
import paper_1901_00913_b200 as kb
import fused_cases as FC
from oracle import kronblur_port as port
from paper_1901_00913_b200.device import DeviceOperator
rng = np.random.default_rng(11)
only = int(sys.argv[1]) if len(sys.argv) > 1 else -1
for i, (m, n, psf, r, bc) in enumerate(FC.cases(rng)):
    if only >= 0 and i != only:
        continue
    op = kb.decompose(psf, kb.BoundaryCondition(bc), s=r, shape=(m, n))
    X = rng.standard_normal((m, n)).astype(np.float32).astype(np.float64)
    dev = DeviceOperator([op], "float32")
    print("case", i, (m, n, psf.values.shape, r, bc), dev.info(), flush=True)
    Xd = torch.from_numpy(X).float().cuda()
    pop = port.PortOperator(op)
    for adj in (False, True):
        y = dev.apply(Xd, adjoint=adj); torch.cuda.synchronize()
        ref = (port.kron_apply_adjoint if adj else port.kron_apply)(pop, X)
        print("  adj" if adj else "  fwd", float(np.linalg.norm(y.double().cpu().numpy() - ref) / np.linalg.norm(ref)), flush=True)
