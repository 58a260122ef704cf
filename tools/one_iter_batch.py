"""A few plain-launched sFISTA iterations of the batch config (cfg3: 512 x 512^2, per-image PSFs)
for ncu captures: python tools/one_iter_batch.py [float32|float64] [iters] [images]
Kernels per iteration: split (forward), sum (residual), split (adjoint), sum (update)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1901_00913_b200 as kb
from paper_1901_00913_b200 import workloads as W
from paper_1901_00913_b200.device import DeviceOperator
from paper_1901_00913_b200.solvers import momentum_table

dtype = sys.argv[1] if len(sys.argv) > 1 else "float32"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 3
images = int(sys.argv[3]) if len(sys.argv) > 3 else 512
cfg = W.CONFIGS["cfg3"]
Bs, ops = [], []
for i in range(images):
    _, psf, B = W.make_image_data(cfg, seed=0, index=i, device="cuda")
    ops.append(kb.decompose(psf, kb.BoundaryCondition(cfg.bc), s=cfg.r, shape=(cfg.m, cfg.m)))
    Bs.append(B)
dev = DeviceOperator(ops, dtype)
Bd = torch.from_numpy(np.stack(Bs)).to("cuda", dev.tdtype)
Xd = torch.zeros_like(Bd)
Yd = torch.zeros_like(Bd)
flag = torch.full((1,), 2**31 - 1, dtype=torch.int32, device="cuda")
_, beta = momentum_table(iters + 1)
dev.sfista_run(Bd, Xd, Yd, beta, 0, iters, np.ones(images), cfg.lam, True, flag, use_graph=False)
torch.cuda.synchronize()
print("ok", dtype, iters, images, float(Xd.double().abs().sum()))
