"""One-sweep tcgen05 kernel (csrc/kb_fused.cuh) against the CPU oracles.

The fused policy is fixed per process (KB_FUSED), so the cases run in a child process with
KB_FUSED=1, which puts every fp32 application the kernel can take on it whatever the image size;
`kb_last_engines` proves which ran. Tolerances: applications within 1e-5 relative Frobenius of
the fp64 oracle; 30-iteration projected solves within 1e-4 and 0.01 dB PSNR of the C oracle
(north_star), L within 1e-5. The default policy at full size is covered by test_gpu_fullsize.py.
"""

import json
import os
import subprocess
import sys

import pytest

from conftest import cuda_ok

pytestmark = pytest.mark.gpu

if not cuda_ok():  # pragma: no cover - collected on CPU but skipped
    pytest.skip("needs a CUDA device", allow_module_level=True)

HERE = os.path.dirname(os.path.abspath(__file__))
FUSED = ["tcgen05_fused"] * 4


@pytest.fixture(scope="module")
def forced():
    env = dict(os.environ, KB_FUSED="1")
    out = subprocess.run([sys.executable, os.path.join(HERE, "fused_cases.py")], env=env, capture_output=True,
                         text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-3000:]
    return [json.loads(line) for line in out.stdout.splitlines() if line.startswith("{")]


def test_fused_operator_parity(forced):
    cases = [c for c in forced if "case" in c]
    assert len(cases) == 10
    for c in cases:
        m, n, shape, r, bc = c["case"]
        if bc == "reflective" and c["engines"][2] != "tcgen05_fused":
            # non-symmetric reflective generators: the adjoint needs the exact folds (two-sweep)
            assert c["engines"][:2] == ["tcgen05_fused"] * 2, c
        else:
            assert c["engines"] == FUSED, c
        assert c["fwd"] <= 1e-5, c
        assert c["adj"] <= 1e-5, c


def test_fused_projected_solve(forced):
    solves = [c for c in forced if "solve" in c]
    assert {c["solve"] for c in solves} == {"zero", "reflective"}
    for c in solves:
        assert c["engines"] == FUSED, c
        assert c["rel"] <= 1e-4, c
        assert c["dpsnr"] <= 0.01, c
        assert c["L_rel"] <= 1e-5, c


def test_fused_batch(forced):
    rows = [c for c in forced if "batch" in c]
    assert {c["batch"] for c in rows} == {"fwd", "adj"}
    for c in rows:
        assert c["rel"] <= 1e-5, c
    eng = [c for c in forced if "batch_engines" in c]
    assert eng and eng[0]["batch_engines"] == FUSED, eng
