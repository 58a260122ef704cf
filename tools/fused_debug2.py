"""One fused apply: python tools/fused_debug2.py m n psf r bc [seed] (KB_FUSED=1)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np, torch
import paper_1901_00913_b200 as kb
from conftest import random_psf
from oracle import kronblur_port as port
from paper_1901_00913_b200.device import DeviceOperator
m, n, w, r = (int(v) for v in sys.argv[1:5]); bc = sys.argv[5]
rng = np.random.default_rng(int(sys.argv[6]) if len(sys.argv) > 6 else 1)
op = kb.decompose(random_psf(rng, w), kb.BoundaryCondition(bc), s=r, shape=(m, n))
X = rng.standard_normal((m, n)).astype(np.float32).astype(np.float64)
dev = DeviceOperator([op], "float32")
Xd = torch.from_numpy(X).float().cuda()
pop = port.PortOperator(op)
for adj in (False, True):
    try:
        y = dev.apply(Xd, adjoint=adj); torch.cuda.synchronize()
    except Exception as ex:
        print(sys.argv[1:], "adj" if adj else "fwd", "FAIL", str(ex).splitlines()[0][-60:], flush=True); sys.exit(1)
    ref = (port.kron_apply_adjoint if adj else port.kron_apply)(pop, X)
    print(sys.argv[1:], "adj" if adj else "fwd", float(np.linalg.norm(y.double().cpu().numpy() - ref) / np.linalg.norm(ref)), flush=True)
