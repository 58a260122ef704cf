"""Dump the Z^T workspace planes after one forward application (debugging the split passes).

usage: tc_zdump.py OUT.npy [m] [w] [r] [bc]
"""
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_1901_00913_b200 as kb
from paper_1901_00913_b200.device import DeviceOperator
sys.path.insert(0, "tests")
from conftest import random_psf
out = sys.argv[1]
m = int(sys.argv[2]) if len(sys.argv) > 2 else 192
w = int(sys.argv[3]) if len(sys.argv) > 3 else 127
r = int(sys.argv[4]) if len(sys.argv) > 4 else 4
bc = sys.argv[5] if len(sys.argv) > 5 else "reflective"
rng = np.random.default_rng(0)
op = kb.decompose(random_psf(rng, w), kb.BoundaryCondition(bc), s=r, shape=(m, m))
X = torch.from_numpy(rng.standard_normal((m, m))).float().cuda()
dev = DeviceOperator([op], "float32")
dev.apply(X)
torch.cuda.synchronize()
b_dlo, b_w = dev.bands[2], dev.bands[3]
H = max(abs(b_dlo), abs(b_dlo + b_w - 1))  # Hb: halo rows of the Z^T planes
rows = m + 2 * H
print("Hb", H, "bands", dev.bands)
z = dev.work.view(torch.float32)[: r * rows * m].view(r, rows, m).cpu().numpy()
np.save(out, z)
print("saved", z.shape)
