"""tcgen05 fp32 passes (csrc/kb_tc.cuh) against the CPU oracle.

The fp32 engine policy is fixed per process (KB_FP32_TC), so the cases run in a child process
with KB_FP32_TC=1, which puts every fp32 pass of an aligned shape on the tcgen05 kernels;
`kb_last_engines` proves they ran there. Tolerances: operator applications within 1e-5 relative
Frobenius of the fp64 oracle; a 30-iteration projected solve within 1e-4 and 0.01 dB PSNR
(north_star). The default policy (wide bands only) is covered at full size by
test_gpu_configs.py and by the engine check below.
"""

import json
import os
import subprocess
import sys

import numpy as np
import pytest

from conftest import cuda_ok

pytestmark = pytest.mark.gpu

if not cuda_ok():  # pragma: no cover - collected on CPU but skipped
    pytest.skip("needs a CUDA device", allow_module_level=True)

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module")
def forced():
    env = dict(os.environ, KB_FP32_TC="1")
    out = subprocess.run([sys.executable, os.path.join(HERE, "tc_cases.py")], env=env, capture_output=True,
                         text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-3000:]
    return [json.loads(line) for line in out.stdout.splitlines() if line.startswith("{")]


def test_tc_operator_parity(forced):
    cases = [c for c in forced if "case" in c]
    assert len(cases) == 9
    for c in cases:
        assert c["engines"] == ["tcgen05_tf32"] * 4, c
        assert c["fwd"] <= 1e-5, c
        assert c["adj"] <= 1e-5, c


def test_tc_projected_solve(forced):
    solves = [c for c in forced if "solve" in c]
    assert {c["solve"] for c in solves} == {"zero", "reflective"}
    for c in solves:
        assert c["rel"] <= 1e-4, c
        assert c["dpsnr"] <= 0.01, c


def test_default_policy_takes_tcgen05_for_wide_bands():
    # 1024^2, w=127, zero BC: Kw = 128 >= both thresholds and 128 chunks -> all four passes on
    # tcgen05; the fp32 result agrees with the fp64 DMMA path
    import torch

    import paper_1901_00913_b200 as kb
    from conftest import random_psf
    from paper_1901_00913_b200.device import DeviceOperator

    if os.environ.get("KB_FP32_TC") is not None:
        pytest.skip("engine policy forced by the environment")
    rng = np.random.default_rng(3)
    m = 1024
    op = kb.decompose(random_psf(rng, 127), kb.BoundaryCondition.ZERO, s=4, shape=(m, m))
    X = torch.from_numpy(rng.random((m, m))).cuda()
    d32 = DeviceOperator([op], "float32")
    d32.time_passes(X.float(), X.float(), 1.0, 0.01, reps=1)
    assert d32.last_engines() == ["tcgen05_tf32"] * 4
    d64 = DeviceOperator([op], "float64")
    for adjoint in (False, True):
        a = d32.apply(X.float(), adjoint=adjoint).double()
        b = d64.apply(X, adjoint=adjoint)
        assert float(torch.linalg.norm(a - b) / torch.linalg.norm(b)) <= 1e-5


@pytest.fixture(scope="module", params=["1", "2"])
def forced_sum1(request):
    # the 128-output sum pass (kb_tc1.cuh) on every tcgen05 sum of tc_cases.py: one accumulator
    # per chunk (KB_TC_SUM1=1) or two (=2) -- small images, wide bands, both BCs, and the exact
    # adjoint fold corrections of non-symmetric reflective generators, none of which the default
    # policy routes through it
    env = dict(os.environ, KB_FP32_TC="1", KB_TC_SUM1=request.param)
    out = subprocess.run([sys.executable, os.path.join(HERE, "tc_cases.py")], env=env, capture_output=True,
                         text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-3000:]
    return [json.loads(line) for line in out.stdout.splitlines() if line.startswith("{")]


def test_single_accumulator_sum_pass_parity(forced_sum1):
    cases = [c for c in forced_sum1 if "case" in c]
    assert len(cases) == 9
    for c in cases:
        assert c["engines"] == ["tcgen05_tf32"] * 4, c
        assert c["fwd"] <= 1e-5, c
        assert c["adj"] <= 1e-5, c
    for c in (c for c in forced_sum1 if "solve" in c):
        assert c["rel"] <= 1e-4, c
        assert c["dpsnr"] <= 0.01, c
