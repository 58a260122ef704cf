"""Device time of the exact blur (kb_blur_direct) at a BASELINE config: python tools/time_blur.py cfg4"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1901_00913_b200 as kb
from paper_1901_00913_b200 import workloads as W

cfg = W.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg4"]
psf = W.make_psf(cfg)
X = torch.rand((cfg.m, cfg.m), device="cuda", dtype=torch.float64)
bc = kb.BoundaryCondition(cfg.bc)
kb.blur_direct(psf, X, bc)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
reps = 3
for _ in range(reps):
    kb.blur_direct(psf, X, bc)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
nnz = int(np.count_nonzero(psf.values))
macs = nnz * cfg.m * cfg.m
print(f"{sys.argv[1] if len(sys.argv) > 1 else 'cfg4'}: {cfg.m}^2, PSF {psf.values.shape} nnz {nnz}: {ms:.1f} ms, "
      f"{2 * macs / ms / 1e9:.2f} TFLOP/s (separately rounded fp64 mul + add)")
