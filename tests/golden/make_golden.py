"""Generate the golden fixtures of tests/golden/ by running the REFERENCE package itself.

Run in the build container (where /root/reference exists):

    cp -r /root/reference/pkg /tmp/refpkg
    PYTHONPATH=/tmp/refpkg/src:. python tests/golden/make_golden.py

Every array here comes from kronblur (the reference) except where noted: the projected solves use
the reference's own kron_apply / kron_apply_adjoint / momentum_next inside a restatement of
solvers._engine with np.maximum(x, 0) after line 171 (the reference has no projection);
without the clamp that restatement reproduces kronblur.sfista bit for bit (checked below).
Full-size fixtures of the BASELINE configs (cfg2-cfg5) come from tests/golden/make_fullsize.py
(the C restatement oracle/kb_oracle.c, itself pinned to these reference fixtures by
tests/test_oracle_c.py), not from this script.
"""

from __future__ import annotations

import decimal
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import kronblur as ref  # noqa: E402
from kronblur import solvers as ref_solvers  # noqa: E402


def engine_projected(op, B, L, lam, iters, project=True):
    """solvers._engine (153-199) with x = max(x, 0) after :171, using reference pieces."""
    b = np.asarray(B, dtype=float)
    x_prev = np.zeros_like(b)
    denom = L + lam**2
    y = x_prev
    t = 1.0
    its = []
    for _ in range(iters):
        grad = ref.kron_apply_adjoint(op, ref.kron_apply(op, y) - b)
        x = (L * y - grad) / denom
        if project:
            x = np.maximum(x, 0.0)
        t_next = ref.momentum_next(t)
        y = x + ((t - 1.0) / t_next) * (x - x_prev)
        its.append(x.copy())
        x_prev = x
        t = t_next
    return x_prev, its


def op_arrays(op):
    return {
        "sigma": np.asarray(op.sigma),
        "rank": np.int64(op.rank),
        "H_c": np.stack([t.H.c for t in op.terms]),
        "K_c": np.stack([t.K.c for t in op.terms]),
        "H_j": np.int64(op.terms[0].H.j),
        "K_j": np.int64(op.terms[0].K.j),
        "kind": np.array(op.terms[0].H.kind.value),
    }


def momentum_decimal(n):
    decimal.getcontext().prec = 60
    t = decimal.Decimal(1)
    out = []
    for _ in range(n):
        t = (1 + (1 + 4 * t * t).sqrt()) / 2
        out.append(float(t))
    return np.array(out)


def main():
    rng = np.random.default_rng(20240817)
    out = {}

    # --- structured.py worked examples and random layouts (test_structured.py:21-87)
    c = np.arange(1.0, 8.0)
    out["toep_c1to7_j4"] = ref.factor_to_dense(ref.toep(c, 4))
    out["hank_c1to7_j3"] = ref.factor_to_dense(ref.hank(c, 3))
    for i in range(12):
        n = int(rng.integers(1, 40))
        j = int(rng.integers(1, n + 1))
        cc = rng.integers(-9, 10, size=n).astype(float)
        out[f"rand{i}_n_j"] = np.array([n, j])
        out[f"rand{i}_c"] = cc
        out[f"rand{i}_T"] = ref.factor_to_dense(ref.toep(cc, j))
        out[f"rand{i}_H"] = ref.factor_to_dense(ref.hank(cc, j))
        out[f"rand{i}_TH"] = ref.factor_to_dense(ref.toep_plus_hank(cc, j))
    for i, (n, j) in enumerate([(150, 60), (257, 129), (1024, 700)]):  # FFT path (n >= 128)
        cc = rng.standard_normal(n)
        X = rng.standard_normal((n, 3))
        out[f"fft{i}_n_j"] = np.array([n, j])
        out[f"fft{i}_c"] = cc
        out[f"fft{i}_X"] = X
        for kind, make in (("T", ref.toep), ("H", ref.hank), ("TH", ref.toep_plus_hank)):
            f = make(cc, j)
            out[f"fft{i}_{kind}_FX"] = ref.factor_apply(f, X)
            out[f"fft{i}_{kind}_FtX"] = ref.factor_apply(f, X, mode="left_transpose")
    np.savez_compressed(os.path.join(HERE, "structured.npz"), **out)

    # --- momentum (test_solvers.py:37-58 uses the first 5 of these, 60-digit)
    ts = []
    t = 1.0
    for _ in range(300):
        t = ref.momentum_next(t)
        ts.append(t)
    np.savez_compressed(os.path.join(HERE, "momentum.npz"), t_ref=np.array(ts),
                        t_decimal=momentum_decimal(300))

    # --- KPA + operator application + Lipschitz + sFISTA on small problems
    out = {}
    cases = [("zero", 5, 16, 3), ("reflective", 5, 16, 3), ("zero", 9, 64, 4),
             ("reflective", 9, 64, 4), ("zero", 31, 96, 3), ("reflective", 15, 80, 5)]
    for ci, (bc, size, m, s) in enumerate(cases):
        rng = np.random.default_rng([20240817, ci])  # per case, so inputs are regenerable
        vals = rng.random((size, size)) + 0.05
        vals /= vals.sum()
        center = (int(rng.integers(1, size + 1)), int(rng.integers(1, size + 1)))
        psf = ref.Psf(vals, center)
        op = ref.decompose(psf, ref.BoundaryCondition(bc), s=s, shape=(m, m))
        X = rng.standard_normal((m, m))
        pre = f"c{ci}_"
        out[pre + "bc"] = np.array(bc)
        out[pre + "psf"] = vals
        out[pre + "center"] = np.array(center)
        out[pre + "m_s"] = np.array([m, s])
        for k, v in op_arrays(op).items():
            out[pre + k] = v
        out[pre + "X"] = X
        out[pre + "AX"] = ref.kron_apply(op, X)
        out[pre + "AtX"] = ref.kron_apply_adjoint(op, X)
        full = ref.decompose(psf, ref.BoundaryCondition(bc), shape=(m, m))
        if m <= 64:
            out[pre + "blur"] = ref.blur_direct(ref.pad_to(psf, m, m), X, ref.BoundaryCondition(bc))
            out[pre + "Afull_X"] = ref.kron_apply(full, X)
        L_mat = ref.estimate_lipschitz(lambda V: ref.kron_apply(op, V),
                                       lambda V: ref.kron_apply_adjoint(op, V), (m, m), 50, ci)
        L_vec = ref.estimate_lipschitz(
            lambda v: ref.vec(ref.kron_apply(op, ref.unvec(v, m, m))),
            lambda v: ref.vec(ref.kron_apply_adjoint(op, ref.unvec(v, m, m))), m * m, 50, ci)
        out[pre + "L_mat"] = np.float64(L_mat)
        out[pre + "L_vec"] = np.float64(L_vec)
        B = ref.kron_apply(op, np.abs(X)) + 0.01 * rng.standard_normal((m, m))
        out[pre + "B"] = B
        iters = 40
        cfg = ref.SolveConfig(lam=0.05, lipschitz=L_mat, max_iter=iters, record_history=False)
        run = ref.sfista(op, B, cfg)
        x_unproj, _ = engine_projected(op, B, L_mat, 0.05, iters, project=False)
        assert np.array_equal(run.x, x_unproj), "restated engine must reproduce sfista exactly"
        out[pre + "x_sfista"] = run.x
        out[pre + "x_proj"], _ = engine_projected(op, B, L_mat, 0.05, iters, project=True)
    np.savez_compressed(os.path.join(HERE, "kron_small.npz"), **out)

    # --- BASELINE cfg1 at full size (the reference's own CPU-runnable config)
    from paper_1901_00913_b200 import workloads as W  # data generation only (host setup)

    cfg = W.CONFIGS["cfg1"]
    Xt, psf_m, B = W.make_image_data(cfg, seed=0, device="cpu")
    psf = ref.Psf(psf_m.values, psf_m.center)
    op = ref.decompose(psf, ref.BoundaryCondition(cfg.bc), s=cfg.r, shape=(cfg.m, cfg.m))
    L = ref.estimate_lipschitz(lambda V: ref.kron_apply(op, V),
                               lambda V: ref.kron_apply_adjoint(op, V), (cfg.m, cfg.m), 50, 0)
    x_proj, _ = engine_projected(op, B, L, cfg.lam, cfg.iters, project=True)
    run = ref.sfista(op, B, ref.SolveConfig(lam=cfg.lam, lipschitz=L, max_iter=cfg.iters,
                                            record_history=False))
    cfg1 = {"B": B, "L": np.float64(L), "x_proj": x_proj, "x_sfista": run.x}
    for k, v in op_arrays(op).items():
        cfg1[k] = v
    np.savez_compressed(os.path.join(HERE, "cfg1.npz"), **cfg1)
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
