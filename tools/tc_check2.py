import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_1901_00913_b200 as kb
from oracle import kronblur_port as port
sys.path.insert(0, "tests")
from conftest import random_psf
for (m, size, s, bc) in [(192,127,4,"zero"),(256,127,4,"reflective"),(192,127,3,"reflective"),(192,63,4,"reflective"),(384,127,4,"reflective"),(192,127,4,"reflective")]:
    rng = np.random.default_rng(0)
    op = kb.decompose(random_psf(rng, size), kb.BoundaryCondition(bc), s=s, shape=(m, m))
    X = rng.standard_normal((m, m))
    pop = port.PortOperator(op)
    want = port.kron_apply(pop, X)
    got = kb.kron_apply(op, X, dtype="float32")
    err = np.abs(got - want)
    rel = np.linalg.norm(got - want) / np.linalg.norm(want)
    bad = np.argwhere(err > 1e-3 * np.abs(want).max())
    print(m, size, s, bc, "fwd rel %.2e" % rel, "bad", len(bad), bad[:3].tolist(), bad[-3:].tolist() if len(bad) else "", flush=True)
