"""Run a few sFISTA iterations of a BASELINE config for ncu captures (no timing)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

import paper_1901_00913_b200 as kb
from paper_1901_00913_b200 import workloads as W
from paper_1901_00913_b200.device import INT_MAX, device_operator

p = argparse.ArgumentParser()
p.add_argument("--config", default="cfg2")
p.add_argument("--dtype", default="float64")
p.add_argument("--iters", type=int, default=3)
p.add_argument("--m", type=int, default=None)
a = p.parse_args()
cfg = W.CONFIGS[a.config]
m = a.m or cfg.m
X, psf, B = W.make_image_data(cfg, seed=0, device="cuda", m=m)
op = kb.decompose(psf, kb.BoundaryCondition(cfg.bc), s=cfg.r, shape=(m, m))
dev = device_operator(op, a.dtype)
_, beta = kb.momentum_table(a.iters)
Bd = torch.from_numpy(B).to("cuda", dev.tdtype)
Xd, Yd = torch.zeros_like(Bd), torch.zeros_like(Bd)
flag = torch.full((1,), INT_MAX, dtype=torch.int32, device="cuda")
dev.sfista_run(Bd, Xd, Yd, beta, 0, a.iters, 1.0, cfg.lam, True, flag, use_graph=False)
torch.cuda.synchronize()
print("ok", float(Xd.abs().max()))
