"""Golden fixtures for the exact blur (tests/golden/blur.npz) from the REFERENCE's blur_direct
(psf.py:170-193). Run in the build container:

    cp -r /root/reference/pkg /tmp/refpkg
    PYTHONPATH=/tmp/refpkg/src:. python tests/golden/make_golden_blur.py

Cases: odd / even / rectangular PSFs, off-centre and corner centres, PSFs with all-zero border
rows and columns, a PSF as large as the image, a 1x1 PSF, rectangular images, both boundary
conditions, and a wide PSF (> 512 columns: the kernel's column-chunk path).
"""

from __future__ import annotations

import os

import numpy as np

import kronblur as ref

HERE = os.path.dirname(os.path.abspath(__file__))

CASES = [  # (m, n, rows, cols, centre or None = random, zero border)
    (16, 16, 5, 5, None, False),
    (33, 20, 7, 4, None, False),
    (40, 57, 9, 9, (1, 1), False),
    (40, 57, 9, 9, (9, 9), False),
    (24, 24, 24, 24, None, False),
    (31, 17, 1, 1, (1, 1), False),
    (64, 48, 15, 11, None, True),
    (20, 40, 6, 10, (3, 8), False),
    (12, 600, 3, 530, (2, 200), False),
]


def main():
    rng = np.random.default_rng(20261020)
    out = {}
    for ci, (m, n, rows, cols, center, border) in enumerate(CASES):
        vals = rng.random((rows, cols)) + 0.05
        if border:
            vals[:2, :] = 0.0
            vals[:, -3:] = 0.0
            vals[5, :] = 0.0
        vals /= vals.sum()
        if center is None:
            center = (int(rng.integers(1, rows + 1)), int(rng.integers(1, cols + 1)))
        psf = ref.Psf(vals, center)
        X = rng.standard_normal((m, n))
        for bc in ("zero", "reflective"):
            pre = f"b{ci}_{bc}_"
            out[pre + "Y"] = ref.blur_direct(psf, X, ref.BoundaryCondition(bc))
        out[f"b{ci}_psf"] = psf.values
        out[f"b{ci}_center"] = np.array(psf.center)
        out[f"b{ci}_X"] = X
    out["ncases"] = np.array(len(CASES))
    np.savez_compressed(os.path.join(HERE, "blur.npz"), **out)
    print("wrote", len(out), "arrays")


if __name__ == "__main__":
    main()
