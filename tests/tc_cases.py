"""Parity cases for the tcgen05 fp32 passes, run in a child process (see test_gpu_tc.py).

The engine policy is read once per process from KB_FP32_TC, so the tests start this module with
KB_FP32_TC=1 (every fp32 pass of an aligned shape on tcgen05) and compare against the CPU oracle.
Prints one JSON object per case.
"""

import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, HERE)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1901_00913_b200 as kb  # noqa: E402
from conftest import random_psf  # noqa: E402
from oracle import kronblur_port as port  # noqa: E402
from paper_1901_00913_b200.device import DeviceOperator  # noqa: E402

# (m, n, psf size, r, bc): zero and reflective, ragged chunks (m % 64 != 0),
# partial 128-column L-tiles, halos wider than half the image (Hb > n / 2)
APPLY = [(64, 64, 9, 3, "zero"), (200, 200, 15, 4, "zero"), (96, 96, 63, 5, "zero"),
         (512, 512, 127, 2, "zero"), (128, 128, 31, 3, "reflective"), (256, 256, 63, 5, "reflective"),
         (192, 192, 127, 4, "reflective"), (300, 300, 33, 6, "reflective"), (136, 136, 41, 8, "reflective")]


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a, np.float64) - b) / np.linalg.norm(b))


def psnr(x, ref):
    mse = float(np.mean((np.asarray(x, np.float64) - ref) ** 2))
    return 10.0 * np.log10(float(np.max(ref)) ** 2 / mse)


def main():
    rng = np.random.default_rng(5)
    for (m, n, size, r, bc) in APPLY:
        op = kb.decompose(random_psf(rng, size), kb.BoundaryCondition(bc), s=r, shape=(m, n))
        X = rng.standard_normal((m, n))
        pop = port.PortOperator(op)
        fwd = rel(kb.kron_apply(op, X, dtype="float32"), port.kron_apply(pop, X))
        adj = rel(kb.kron_apply_adjoint(op, X, dtype="float32"), port.kron_apply_adjoint(pop, X))
        dev = DeviceOperator([op], "float32")
        Xd = torch.from_numpy(X).float().cuda()
        dev.time_passes(Xd, Xd, 1.0, 0.01, reps=1)
        print(json.dumps({"case": [m, n, size, r, bc], "fwd": fwd, "adj": adj,
                          "engines": dev.last_engines()}), flush=True)
    # a projected solve (residual + fused update + power-iteration Lipschitz on tcgen05)
    m, size, r = 256, 63, 4
    for bc in ("zero", "reflective"):
        X0 = np.clip(rng.random((m, m)) - 0.3, 0, None)
        op = kb.decompose(random_psf(rng, size), kb.BoundaryCondition(bc), s=r, shape=(m, m))
        B = port.kron_apply(port.PortOperator(op), X0)
        B = (B + 0.01 * np.linalg.norm(B) / m * rng.standard_normal(B.shape)).astype(np.float32).astype(np.float64)
        L = kb.lipschitz(op, iters=30, seed=0)
        want, _ = port.sfista(op, B, L, 0.02, 30, project=True)
        got = kb.sfista(op, B, kb.SolveConfig(lam=0.02, lipschitz=L, max_iter=30, record_history=False),
                        options=kb.SolveOptions(dtype="float32", project=True)).x
        print(json.dumps({"solve": bc, "rel": rel(got, want), "dpsnr": abs(psnr(got, X0) - psnr(want, X0))}),
              flush=True)


if __name__ == "__main__":
    main()
