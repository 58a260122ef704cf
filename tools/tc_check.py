import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_1901_00913_b200 as kb
from oracle import kronblur_port as port
sys.path.insert(0, "tests")
from conftest import random_psf
rng = np.random.default_rng(0)
cases = [(64, 9, 3, "zero"), (256, 31, 3, "zero"), (200, 15, 4, "zero"), (96, 63, 5, "zero"),
         (512, 127, 2, "zero"), (128, 31, 3, "reflective"), (256, 63, 5, "reflective"),
         (192, 127, 4, "reflective"), (300, 33, 6, "reflective")]
for (m, size, s, bc) in cases:
    op = kb.decompose(random_psf(rng, size), kb.BoundaryCondition(bc), s=s, shape=(m, m))
    X = rng.standard_normal((m, m))
    pop = port.PortOperator(op)
    want = port.kron_apply(pop, X)
    got = kb.kron_apply(op, X, dtype="float32")
    wantT = port.kron_apply_adjoint(pop, X)
    gotT = kb.kron_apply_adjoint(op, X, dtype="float32")
    rel = np.linalg.norm(got - want) / np.linalg.norm(want)
    relT = np.linalg.norm(gotT - wantT) / np.linalg.norm(wantT)
    print(m, size, s, bc, "fwd rel %.2e  adj rel %.2e" % (rel, relT), flush=True)
