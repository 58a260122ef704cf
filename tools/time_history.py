"""Wall time of a record_history=True sfista solve (the reference's default SolveConfig) at a
BASELINE config, against the history-free fast path: python tools/time_history.py [cfg] [iters]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_1901_00913_b200 as kb
from paper_1901_00913_b200 import workloads as W

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 200
cfg = W.CONFIGS[name]
X, psf, B = W.make_image_data(cfg, seed=0, device="cuda")
op = kb.decompose(psf, kb.BoundaryCondition(cfg.bc), s=cfg.r, shape=(cfg.m, cfg.m))
for hist in (False, True, True):
    c = kb.SolveConfig(lam=cfg.lam, lipschitz=1.0, max_iter=iters, record_history=hist)
    t0 = time.perf_counter()
    run = kb.sfista(op, B, c, truth=X if hist else None)
    wall = time.perf_counter() - t0
    print(f"{name} record_history={hist}: wall {wall * 1e3:.1f} ms, solve_ms {run.solve_ms:.1f}, "
          f"{len(run.history)} records, last objective {run.history[-1].objective if hist else float('nan'):.6e}")
