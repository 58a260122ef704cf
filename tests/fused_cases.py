"""Parity cases for the one-sweep tcgen05 kernel (csrc/kb_fused.cuh), run in a child process.

The fused policy is read once per process from KB_FUSED, so test_gpu_fused.py starts this module
with KB_FUSED=1 (every fp32 application the kernel can take runs fused, whatever its size) and
compares with the CPU oracles. Prints one JSON object per case.
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
from oracle import kb_oracle as C  # noqa: E402
from oracle import kronblur_port as port  # noqa: E402
from paper_1901_00913_b200 import workloads as W  # noqa: E402
from paper_1901_00913_b200.device import DeviceOperator  # noqa: E402


def sym_psf(w, s1, s2, ang):
    """rotated Gaussian: point-symmetric, so the reflective adjoint takes the fused sign fills"""
    return kb.Psf(W._rot_gauss(w, s1, s2, ang), ((w + 1) // 2, (w + 1) // 2))


# (m, n, psf, r, bc): one tile and ragged tiles (m % 128, n % 16), partial column chunks, halos
# wider than a chunk, both BCs, symmetric and non-symmetric generators (the non-symmetric
# reflective adjoint needs the exact folds and stays on the two-sweep passes), r up to 10,
# many tiles per CTA
def cases(rng):
    return [
        (64, 64, random_psf(rng, 9), 3, "zero"),
        (200, 200, random_psf(rng, 15), 4, "zero"),
        (256, 256, sym_psf(31, 4.0, 1.5, 0.5), 3, "reflective"),
        (300, 300, sym_psf(33, 5.0, 2.0, 1.1), 6, "reflective"),
        (136, 136, sym_psf(41, 6.0, 3.0, 0.3), 8, "reflective"),
        (512, 512, sym_psf(63, 9.0, 4.0, 0.9), 5, "reflective"),
        (384, 384, sym_psf(57, 8.0, 2.5, 2.0), 10, "reflective"),
        (260, 260, random_psf(rng, 31, 17), 5, "zero"),
        (192, 192, random_psf(rng, 25), 4, "reflective"),
        (896, 896, sym_psf(29, 3.0, 3.0, 0.0), 4, "zero"),
    ]


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a, np.float64) - b) / np.linalg.norm(b))


def psnr(x, ref):
    mse = float(np.mean((np.asarray(x, np.float64) - ref) ** 2))
    return 10.0 * np.log10(float(np.max(ref)) ** 2 / mse)


def main():
    rng = np.random.default_rng(11)
    for (m, n, psf, r, bc) in cases(rng):
        op = kb.decompose(psf, kb.BoundaryCondition(bc), s=r, shape=(m, n))
        X = rng.standard_normal((m, n)).astype(np.float32).astype(np.float64)
        pop = port.PortOperator(op)
        dev = DeviceOperator([op], "float32")
        Xd = torch.from_numpy(X).float().cuda()
        fwd = rel(dev.apply(Xd).double().cpu().numpy(), port.kron_apply(pop, X))
        adj = rel(dev.apply(Xd, adjoint=True).double().cpu().numpy(), port.kron_apply_adjoint(pop, X))
        dev.time_passes(Xd, Xd, 1.0, 0.01, reps=1)
        print(json.dumps({"case": [m, n, list(psf.values.shape), r, bc], "fwd": fwd, "adj": adj,
                          "engines": dev.last_engines(), "half_widths": list(dev.half_widths)}), flush=True)
    # projected solves (residual + fused update) and the power iteration against the C oracle
    for bc, m, w, r in (("zero", 256, 31, 4), ("reflective", 384, 45, 6)):
        X0 = np.clip(rng.random((m, m)) - 0.3, 0, None)
        op = kb.decompose(sym_psf(w, 5.0, 2.0, 0.7), kb.BoundaryCondition(bc), s=r, shape=(m, m))
        B = port.kron_apply(port.PortOperator(op), X0)
        B = (B + 0.01 * np.linalg.norm(B) / m * rng.standard_normal(B.shape)).astype(np.float32).astype(np.float64)
        L = kb.lipschitz(op, iters=30, seed=0, dtype="float32")
        pop = port.PortOperator(op)
        L64 = port.estimate_lipschitz(lambda Y: port.kron_apply(pop, Y), lambda Y: port.kron_apply_adjoint(pop, Y),
                                      (m, m), iters=30, seed=0)
        _, beta = kb.momentum_table(30)
        want = C.sfista(C.OracleOp(op, "float32"), B, L, 0.02, 30, beta, project=True)
        run = kb.sfista(op, B, kb.SolveConfig(lam=0.02, lipschitz=L, max_iter=30, record_history=False),
                        options=kb.SolveOptions(dtype="float32", project=True))
        dev = DeviceOperator([op], "float32")
        dev.time_passes(torch.from_numpy(B).float().cuda(), torch.from_numpy(B).float().cuda(), L, 0.02, reps=1)
        print(json.dumps({"solve": bc, "rel": rel(run.x, want), "dpsnr": abs(psnr(run.x, X0) - psnr(want, X0)),
                          "L_rel": abs(L - L64) / L64, "engines": dev.last_engines()}), flush=True)
    # a cfg3-style batch: per-image PSFs, zero BC, one launch over all images
    ops, Xs = [], []
    for k in range(6):
        ops.append(kb.decompose(sym_psf(31, 2.0 + 0.5 * k, 1.2, 0.4 * k), kb.BoundaryCondition.ZERO, s=4,
                                shape=(256, 256)))
        Xs.append(rng.standard_normal((256, 256)).astype(np.float32).astype(np.float64))
    dev = DeviceOperator(ops, "float32")
    Xd = torch.from_numpy(np.stack(Xs)).float().cuda()
    for adjoint in (False, True):
        got = dev.apply(Xd, adjoint=adjoint).double().cpu().numpy()
        fn = port.kron_apply_adjoint if adjoint else port.kron_apply
        worst = max(rel(got[k], fn(port.PortOperator(ops[k]), Xs[k])) for k in range(len(ops)))
        print(json.dumps({"batch": "adj" if adjoint else "fwd", "rel": worst}), flush=True)
    dev.time_passes(Xd, Xd, 1.0, 0.01, reps=1)
    print(json.dumps({"batch_engines": dev.last_engines()}), flush=True)


if __name__ == "__main__":
    main()
