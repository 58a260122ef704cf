"""Where the public sfista() call spends its host time (run on the GPU box):
python tools/e2e_profile.py cfg1 float64 [calls]  -> wall time per call, solve_ms, cProfile top."""
import cProfile
import pstats
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_1901_00913_b200 as kb  # noqa: E402
from paper_1901_00913_b200 import workloads as W  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg1"
dtype = sys.argv[2] if len(sys.argv) > 2 else "float64"
calls = int(sys.argv[3]) if len(sys.argv) > 3 else 50
cfg = W.CONFIGS[name]
B, op, L = bench.build_problem(cfg, dtype)
opts = kb.SolveOptions(dtype=dtype, project=True, use_graph=True)
sc = kb.SolveConfig(lam=cfg.lam, lipschitz=float(L), max_iter=cfg.iters, record_history=False)
for _ in range(3):
    run = kb.sfista(op, B, sc, options=opts)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(calls):
    run = kb.sfista(op, B, sc, options=opts)
torch.cuda.synchronize()
wall = (time.perf_counter() - t0) / calls
print(f"{name} {dtype}: {wall * 1e3:.3f} ms per call, solve_ms {run.solve_ms:.3f}, "
      f"{cfg.m * cfg.m * cfg.iters / 1e6 / wall:.1f} Mpix*it/s e2e")
pr = cProfile.Profile()
pr.enable()
for _ in range(calls):
    kb.sfista(op, B, sc, options=opts)
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(28)
