"""Quick check of the fused kernel on one small case (run with KB_FUSED=1)."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np, torch
import paper_1901_00913_b200 as kb
from conftest import random_psf
from oracle import kronblur_port as port
from paper_1901_00913_b200.device import DeviceOperator
rng = np.random.default_rng(1)
m = int(sys.argv[1]) if len(sys.argv) > 1 else 256
bc = sys.argv[2] if len(sys.argv) > 2 else "zero"
op = kb.decompose(random_psf(rng, 15), kb.BoundaryCondition(bc), s=3, shape=(m, m))
X = rng.standard_normal((m, m)).astype(np.float32).astype(np.float64)
dev = DeviceOperator([op], "float32")
Xd = torch.from_numpy(X).float().cuda()
t = time.time()
y = dev.apply(Xd); torch.cuda.synchronize()
print("apply done", time.time() - t, flush=True)
pop = port.PortOperator(op)
ref = port.kron_apply(pop, X)
print("fwd rel", np.linalg.norm(y.double().cpu().numpy() - ref) / np.linalg.norm(ref), flush=True)
ya = dev.apply(Xd, adjoint=True); torch.cuda.synchronize()
refa = port.kron_apply_adjoint(pop, X)
print("adj rel", np.linalg.norm(ya.double().cpu().numpy() - refa) / np.linalg.norm(refa), flush=True)
dev.time_passes(Xd, Xd, 1.0, 0.01, reps=1)
print("engines", dev.last_engines(), flush=True)
