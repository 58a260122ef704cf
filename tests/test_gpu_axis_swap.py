"""The axis-swapped twin (kb_capi.cu): for large fp32 images whose axis-1 band is markedly wider,
the fast sFISTA path solves the transposed problem Y^T = sum_i K_i X^T H_i^T (the wider band in
pass A). Forced on a small image (KB_AXIS_SWAP=1 is read once per process, so a subprocess runs
it) and off (KB_AXIS_SWAP=0), both against the C oracle; at cfg5 it is the default (the
full-size tests in test_gpu_fullsize.py run it)."""

import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT, cuda_ok

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_ok(), reason="needs a CUDA device")]

SCRIPT = r"""
import json, sys
sys.path.insert(0, ROOT)
import numpy as np
import paper_1901_00913_b200 as kb
from oracle import kb_oracle as C
from paper_1901_00913_b200 import workloads as W
from paper_1901_00913_b200.device import device_operator
out = {}
for bc in ("reflective", "zero"):
    cfg = W.CONFIGS["cfg5"]
    X, psf, B = W.make_image_data(cfg, seed=1, m=512, counts=(200, 100), device="cuda")
    op = kb.decompose(psf, kb.BoundaryCondition(bc), s=6, shape=(512, 512))
    B = B.astype(np.float32).astype(np.float64)
    L = kb.lipschitz(op, iters=30, seed=0)
    run = kb.sfista(op, B, kb.SolveConfig(lam=0.01, lipschitz=L, max_iter=12, record_history=False),
                    options=kb.SolveOptions(dtype="float32", project=True))
    _, beta = kb.momentum_table(12)
    want = C.sfista(C.OracleOp(op, "float32"), B, L, 0.01, 12, beta, project=True)
    dev = device_operator(op, "float32")
    out[bc] = {"rel": float(np.linalg.norm(run.x - want) / np.linalg.norm(want)), "twin": dev.info()["twin"],
               "engines": dev.last_engines()}
print(json.dumps(out))
"""


@pytest.mark.parametrize("swap", ["1", "0"])
def test_axis_swapped_solve_matches_oracle(swap):
    env = dict(os.environ, KB_AXIS_SWAP=swap)
    out = subprocess.run([sys.executable, "-c", f"ROOT = {ROOT!r}\n" + SCRIPT], capture_output=True, text=True,
                         timeout=600, env=env, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    res = json.loads(out.stdout.strip().splitlines()[-1])
    for bc, r in res.items():
        assert r["twin"] == int(swap), (bc, r)
        assert r["rel"] <= 1e-4, (bc, r)
