"""A few plain-launched sFISTA iterations of a BASELINE config (no CUDA graph) for ncu captures.

usage: one_iter.py [float64|float32] [iters] [config, default cfg2]
Each iteration launches kb_pass_split (forward), kb_pass_sum (residual), kb_pass_split
(adjoint), kb_pass_sum (update) in that order; `ncu -k regex:kb_pass_ -s 4 -c 4` captures the
second iteration's four kernels with the first as warm-up.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1901_00913_b200 as kb
from paper_1901_00913_b200 import workloads as W
from paper_1901_00913_b200.device import device_operator
from paper_1901_00913_b200.solvers import momentum_table

dtype = sys.argv[1] if len(sys.argv) > 1 else "float64"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 3
cfg = W.CONFIGS[sys.argv[3] if len(sys.argv) > 3 else "cfg2"]
_, psf, B = W.make_image_data(cfg, seed=0, device="cuda")
op = kb.decompose(psf, kb.BoundaryCondition(cfg.bc), s=cfg.r, shape=(cfg.m, cfg.m))
dev = device_operator(op, dtype)
Bd = torch.from_numpy(B).to("cuda", dev.tdtype)
Xd = torch.zeros_like(Bd)
Yd = torch.zeros_like(Bd)
flag = torch.full((1,), 2**31 - 1, dtype=torch.int32, device="cuda")
_, beta = momentum_table(iters + 1)
dev.sfista_run(Bd, Xd, Yd, beta, 0, iters, 1.0, cfg.lam, True, flag, use_graph=False)
torch.cuda.synchronize()
print("ok", dtype, iters, float(Xd.double().abs().sum()))
