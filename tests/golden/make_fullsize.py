"""Full-size, full-length parity fixtures for BASELINE cfg2-cfg5 (test infrastructure).

The reference's own CPU path cannot run these configs in a test (cfg4 6.4 h, cfg5
~4.5 days per solve), so they are computed offline, once, by the C restatement of the reference
hot path (oracle/kb_oracle.c, OpenMP fp64), which tests/test_oracle_c.py pins to the reference's
own outputs (kron_apply/adjoint, L, projected solves, cfg1 at full size, blur_direct bit for bit).

Each fixture holds what the GPU test needs to rebuild the identical problem and judge the
result, not the full solution (which would be up to 2 GiB):
  * the config, seed, iteration count, lambda and the Lipschitz constant L (the oracle's
    matrix-form 50-step power iteration: both sides get the same float);
  * a fingerprint of the noisy data B (sum and 256 sampled entries) so the test can assert it
    regenerated the same B on the GPU (phantom painting is exact; blur_direct is bit-identical
    on both sides; the noise scale may differ in the last bit between BLAS builds);
  * the oracle's x_iters: every row's 2-norm, the Frobenius norm, sampled full rows, and its
    PSNR against the ground truth (peak 1: intensities are U[0,1]).
fp32 configs feed the oracle the fp32-rounded data and generator taps.

Run here (8 host cores: ~1 h for all five): python tests/golden/make_fullsize.py [cfg ...]
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import paper_1901_00913_b200 as kb  # noqa: E402  (setup code only: phantom, PSF, KPA)
from paper_1901_00913_b200 import workloads as W  # noqa: E402
from oracle import kb_oracle as C  # noqa: E402
from oracle import kronblur_port as port  # noqa: E402

# (config, dtype) -> sampled rows, cfg3 sampled images
CASES = {
    "cfg2_float64": ("cfg2", "float64"),
    "cfg2_float32": ("cfg2", "float32"),
    "cfg3_float32": ("cfg3", "float32"),
    "cfg4_float32": ("cfg4", "float32"),
    "cfg5_float32": ("cfg5", "float32"),
}
CFG3_IMAGES = (0, 1, 63, 127, 255, 300, 411, 511)
SEED = 0


def psnr(x, truth):
    mse = float(np.mean((np.asarray(x, dtype=np.float64) - truth) ** 2))
    return 10.0 * np.log10(1.0 / mse)


def sample_rows(m, count, seed=123):
    rng = np.random.default_rng(seed)
    rest = rng.choice(np.arange(2, m - 2), size=count - 4, replace=False)
    return np.unique(np.concatenate([[0, 1, m // 2, m - 1], rest])).astype(np.int64)


def problem(cfg, index=0):
    """(truth, psf, B) exactly as workloads.make_image_data builds them on the GPU, with the
    exact blur by the C restatement of blur_direct (bit-identical to the reference)."""
    X = W.phantom(cfg.m, cfg.n_rect, cfg.n_disk, SEED * 100003 + index, device="cpu").numpy()
    psf = W.make_psf(cfg, index=index, seed=SEED)
    b = C.blur_direct(psf.values, psf.center, X, cfg.bc)
    B = W.add_noise(b, cfg.noise, SEED * 100003 + index)
    return X, psf, B


def solve_one(cfg, dtype, X, psf, B, rows_count):
    op = kb.decompose(psf, kb.BoundaryCondition(cfg.bc), s=cfg.r, shape=(cfg.m, cfg.m))
    t0 = time.time()
    rho, _ = C.power(C.OracleOp(op), port.lipschitz_start(SEED, (cfg.m, cfg.m)), 50)
    L = 1.05 * float(rho[-1])
    t1 = time.time()
    Bin = B.astype(np.float32).astype(np.float64) if dtype == "float32" else B
    _, beta = kb.momentum_table(cfg.iters)
    x = C.sfista(C.OracleOp(op, dtype), Bin, L, cfg.lam, cfg.iters, beta, project=True)
    t2 = time.time()
    rows = sample_rows(cfg.m, rows_count)
    out = {
        "L": np.float64(L), "lam": np.float64(cfg.lam), "iters": np.int64(cfg.iters),
        "row_norms": np.linalg.norm(x, axis=1), "fro": np.float64(np.linalg.norm(x)),
        "rows_idx": rows, "rows": x[rows].astype(np.float32 if dtype == "float32" else np.float64),
        "psnr": np.float64(psnr(x, X)), "psnr_truth_b": np.float64(psnr(B, X)),
    }
    flat = np.random.default_rng(7).integers(0, B.size, size=256)
    out["b_idx"], out["b_vals"], out["b_sum"] = flat, B.ravel()[flat], np.float64(B.sum())
    print(f"  L={L:.12g} ({t1 - t0:.0f} s)  solve {cfg.iters} it ({t2 - t1:.0f} s)  psnr {out['psnr']:.4f}",
          flush=True)
    return out


def make(case):
    name, dtype = CASES[case]
    cfg = W.CONFIGS[name]
    print(f"{case}: {cfg}", flush=True)
    if cfg.batch > 1:
        out = {"images": np.array(CFG3_IMAGES, dtype=np.int64)}
        for i in CFG3_IMAGES:
            X, psf, B = problem(cfg, i)
            for k, v in solve_one(cfg, dtype, X, psf, B, 8).items():
                out[f"i{i}_{k}"] = v
    else:
        X, psf, B = problem(cfg)
        out = solve_one(cfg, dtype, X, psf, B, 8 if cfg.m >= 16384 else 16)
    out["config"] = np.array(name)
    out["dtype"] = np.array(dtype)
    out["oracle_threads"] = np.int64(C.threads())
    path = os.path.join(HERE, f"full_{case}.npz")
    np.savez_compressed(path, **out)
    print(f"  -> {path} ({os.path.getsize(path) / 1e6:.2f} MB)", flush=True)


if __name__ == "__main__":
    for case in sys.argv[1:] or list(CASES):
        make(case)
