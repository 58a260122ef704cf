"""Per-kernel CUDA-event times of one cfg2 iteration (kb_time_passes), for quick experiments."""
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
X, psf, B = W.make_image_data(cfg, seed=0, device="cuda", m=m, counts=(cfg.n_rect, cfg.n_disk) if m == cfg.m else (50, 25))
op = kb.decompose(psf, kb.BoundaryCondition(cfg.bc), s=cfg.r, shape=(m, m))
dev = device_operator(op, dtype)
Bd = torch.from_numpy(B).to("cuda", dev.tdtype)
ms = dev.time_passes(Bd, Bd, 1.0, cfg.lam, reps=20)
print(name, dtype, m, "KB_DEBUG_MODE=%s" % os.environ.get("KB_DEBUG_MODE", "0"), [round(x * 1000, 1) for x in ms], "us")
