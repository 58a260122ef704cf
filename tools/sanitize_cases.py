"""Tiny invocations of every kernel family, for compute-sanitizer (tests/test_gpu_sanitizer.py).

usage: python tools/sanitize_cases.py FAMILY   (FAMILY in dmma, tf32, tcgen05, ffma, generic,
persist, blur, norms). Engine selection is by shape / dtype / env (KB_FP32_TC, KB_FP32_PATH,
KB_PERSIST are read once per process, so the test runs each family in its own process)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1901_00913_b200 as kb
from paper_1901_00913_b200.device import device_operator

fam = sys.argv[1]
rng = np.random.default_rng(1)
vals = rng.random((9, 7)) + 0.05
psf = kb.Psf(vals / vals.sum(), (5, 3))
shape, dtype = {"dmma": ((128, 96), "float64"), "tf32": ((128, 96), "float32"),
                "tcgen05": ((256, 256), "float32"), "ffma": ((128, 96), "float32"),
                "generic": ((45, 37), "float64"), "persist": ((96, 80), "float64"),
                "blur": ((40, 36), "float64"), "norms": ((64, 64), "float32")}[fam]
if fam == "blur":
    X = rng.random(shape)
    for bc in ("zero", "reflective"):
        kb.blur_direct(psf, X, kb.BoundaryCondition(bc))
    torch.cuda.synchronize()
    print("ok", fam)
    sys.exit(0)
for bc in ("zero", "reflective"):
    op = kb.decompose(psf, kb.BoundaryCondition(bc), s=3, shape=shape)
    X = rng.random(shape)
    kb.kron_apply(op, X, dtype=dtype)
    kb.kron_apply_adjoint(op, X, dtype=dtype)
    L = kb.lipschitz(op, iters=3, seed=0, dtype=dtype)
    cfg = kb.SolveConfig(lam=0.05, lipschitz=L, max_iter=3, record_history=(fam == "norms"))
    run = kb.sfista(op, X, cfg, options=kb.SolveOptions(dtype=dtype, project=True, use_graph=False))
    print(fam, bc, device_operator(op, dtype).last_engines(), float(np.abs(run.x).sum()))
torch.cuda.synchronize()
print("ok", fam)
