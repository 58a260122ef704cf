"""Error of a full-length solve against its committed fixture (tests/golden/full_<case>.npz):
python tools/fullsize_err.py cfg4_float32   -- prints the relative errors the parity test bounds."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
import test_gpu_fullsize as T
f = T.fixture(sys.argv[1])
name, dtype = str(f["config"]), str(f["dtype"])
cfg = T.W.CONFIGS[name]
X, psf, B = T.W.make_image_data(cfg, seed=0, device="cuda")
op = T.kb.decompose(psf, T.kb.BoundaryCondition(cfg.bc), s=cfg.r, shape=(cfg.m, cfg.m))
x, engines = T.solve(op, B, float(f["L"]), cfg, dtype, int(f["iters"]))
rows = f["rows_idx"]
print(sys.argv[1], engines, "rows rel", T.rel(x[rows], f["rows"].astype(np.float64)),
      "row-norm rel", T.rel(np.linalg.norm(x, axis=1), f["row_norms"]),
      "fro rel", abs(float(np.linalg.norm(x)) - float(f["fro"])) / float(f["fro"]),
      "dpsnr", abs(T.psnr(x, X) - float(f["psnr"])), "tol", T.TOL[dtype])
