"""tc1 epilogue debug: one apply (PLAIN), a few sfista iterations (RESID/UPDATE), a power step."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np, torch
import paper_1901_00913_b200 as kb
from conftest import random_psf
from oracle import kronblur_port as port
from paper_1901_00913_b200.device import DeviceOperator
rng = np.random.default_rng(3)
m = int(sys.argv[1]) if len(sys.argv) > 1 else 256
op = kb.decompose(random_psf(rng, 31), kb.BoundaryCondition(os.environ.get("BC", "zero")), s=int(os.environ.get("R", "3")), shape=(m, m))
X = rng.standard_normal((m, m)).astype(np.float32).astype(np.float64)
dev = DeviceOperator([op], "float32")
Xd = torch.from_numpy(X).float().cuda()
pop = port.PortOperator(op)
for what in sys.argv[2:] or ["apply", "power", "solve"]:
    if what == "apply":
        y = dev.apply(Xd); torch.cuda.synchronize()
        ref = port.kron_apply(pop, X)
        print("apply rel", float(np.linalg.norm(y.double().cpu().numpy() - ref) / np.linalg.norm(ref)), flush=True)
    elif what == "power":
        L = kb.lipschitz(op, iters=5, seed=0, dtype="float32"); torch.cuda.synchronize()
        print("power L", L, flush=True)
    else:
        run = kb.sfista(op, X, kb.SolveConfig(lam=0.02, lipschitz=2.0, max_iter=5, record_history=False),
                        options=kb.SolveOptions(dtype="float32", project=True))
        print("solve ok", float(np.abs(run.x).sum()), flush=True)
