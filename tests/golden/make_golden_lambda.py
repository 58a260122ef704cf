"""Golden fixtures for select_lambda (tests/golden/lambda.npz) from the REFERENCE
(solvers.py:255-306), both routes. Run in the build container:

    cp -r /root/reference/pkg /tmp/refpkg
    PYTHONPATH=/tmp/refpkg/src:. python tests/golden/make_golden_lambda.py
"""

from __future__ import annotations

import os

import numpy as np

import kronblur as ref

HERE = os.path.dirname(os.path.abspath(__file__))

CASES = [  # (m, psf size, bc, noise level, L, data): data "rand" = U[0,1) + 0.5 (the reference
    # tests' style), "blur" = blurred U[0,1) image plus Gaussian noise of exactly that level, so the
    # discrepancy target falls inside the residual range and the choice is an interior grid point
    (6, 3, "reflective", 0.0, 1.2, "rand"),     # dense route, noise-free -> smallest grid point
    (6, 3, "reflective", 0.2, 1.2, "rand"),     # dense route
    (30, 3, "zero", 0.05, 1.2, "blur"),         # dense route (900 <= 1024), interior choice
    (34, 3, "reflective", 0.05, 1.1, "blur"),   # probe route (34^2 > 1024)
    (40, 5, "zero", 0.02, None, "blur"),        # probe route, L from the reference power iteration
    (48, 7, "reflective", 0.1, None, "blur"),   # probe route
]


def main():
    rng = np.random.default_rng(1901)
    out = {}
    for ci, (m, k, bc, noise, L, off) in enumerate(CASES):  # noqa: B007
        vals = rng.random((k, k)) + 0.05
        vals /= vals.sum()
        center = (int(rng.integers(1, k + 1)), int(rng.integers(1, k + 1)))
        psf = ref.Psf(vals, center)
        op = ref.decompose(psf, ref.BoundaryCondition(bc), shape=(m, m))
        if off == "rand":
            B = rng.random((m, m)) + 0.5
        else:
            B0 = ref.kron_apply(op, rng.random((m, m)))
            g = rng.standard_normal((m, m))
            B = B0 + noise * np.linalg.norm(B0) / np.linalg.norm(g) * g
        if L is None:
            L = ref.estimate_lipschitz(lambda V: ref.kron_apply(op, V), lambda V: ref.kron_apply_adjoint(op, V),
                                       (m, m), 50, ci)
        lam = ref.select_lambda(op, B, noise, L)
        pre = f"l{ci}_"
        out[pre + "psf"] = vals
        out[pre + "center"] = np.array(center)
        out[pre + "bc"] = np.array(bc)
        out[pre + "B"] = B
        out[pre + "noise_L"] = np.array([noise, L])
        out[pre + "lam"] = np.float64(lam)
    out["ncases"] = np.array(len(CASES))
    np.savez_compressed(os.path.join(HERE, "lambda.npz"), **out)
    print("wrote", len(out), "arrays")


if __name__ == "__main__":
    main()
