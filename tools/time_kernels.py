"""Per-kernel CUDA-event times of one iteration (kb_time_passes), for quick experiments.

usage: time_kernels.py [cfg] [dtype] [m] [r] [bc]   (KB_DEBUG_MODE env selects profiling switches)
"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1901_00913_b200 as kb
from paper_1901_00913_b200 import workloads as W
from paper_1901_00913_b200.device import device_operator
name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
dtype = sys.argv[2] if len(sys.argv) > 2 else "float64"
cfg = W.CONFIGS[name]
m = int(sys.argv[3]) if len(sys.argv) > 3 else cfg.m
r = int(sys.argv[4]) if len(sys.argv) > 4 else cfg.r
bc = sys.argv[5] if len(sys.argv) > 5 else cfg.bc
X, psf, B = W.make_image_data(cfg, seed=0, device="cuda", m=m, counts=(cfg.n_rect, cfg.n_disk) if m == cfg.m else (50, 25))
op = kb.decompose(psf, kb.BoundaryCondition(bc), s=r, shape=(m, m))
dev = device_operator(op, dtype)
Bd = torch.from_numpy(B).to("cuda", dev.tdtype)
ms = dev.time_passes(Bd, Bd, 1.0, cfg.lam, reps=20)
print(name, dtype, m, bc, "r=%d" % len(op.terms), "KB_DEBUG_MODE=%s" % os.environ.get("KB_DEBUG_MODE", "0"),
      [round(x * 1000, 1) for x in ms], "us")
