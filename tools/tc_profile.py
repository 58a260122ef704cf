"""Per-role stall cycles of the tcgen05 split kernel (KB_FP32_TC=1 KB_DEBUG_MODE=128; needs a -DKB_TC_PROF=1 build, e.g. tools/variant.sh prof -DKB_TC_PROF=1).

usage: tc_profile.py [cfg] [m]   -- prints the block-mean of each kb_tc.cuh TcProf slot (kcycles)
"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1901_00913_b200 as kb
from paper_1901_00913_b200 import workloads as W
from paper_1901_00913_b200.device import device_operator, load_library
name = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
cfg = W.CONFIGS[name]
m = int(sys.argv[2]) if len(sys.argv) > 2 else cfg.m
_, psf, B = W.make_image_data(cfg, seed=0, device="cuda", m=m, counts=(cfg.n_rect, cfg.n_disk) if m == cfg.m else (50, 25))
op = kb.decompose(psf, kb.BoundaryCondition("zero"), s=cfg.r, shape=(m, m))
dev = device_operator(op, "float32")
Bd = torch.from_numpy(B).to("cuda", torch.float32)
for _ in range(3):
    dev.apply(Bd)
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * (2 * 1024 * 8))()
assert load_library().kb_debug_trace(buf, 2 * 1024 * 8) == 0
allk = np.frombuffer(buf, dtype=np.uint64).reshape(2, 1024, 8).astype(np.float64)
a = allk[0]
a = a[a[:, 7] > 0]
names = ["converter convert+st", "converter a_free wait", "converter full wait", "converter bricks",
         "epilogue busy", "converter wait::st", "issuer a_ready wait", "converter total"]
print(f"{name} m={m}: {len(a)} blocks")
for i, nm in enumerate(names):
    print(f"  {nm:24s} mean {a[:, i].mean() / 1e3:9.1f} kcyc  max {a[:, i].max() / 1e3:9.1f}")
s = allk[1]
s = s[s[:, 7] > 0]
names1 = ["converter convert+st", "converter a_free wait", "converter full wait", "converter fence+arrives",
          "issuer a_ready wait", "issuer slot/bready wait", "converter wait::st", "converter total"]
print(f"sum pass: {len(s)} blocks")
for i, nm in enumerate(names1):
    if len(s):
        print(f"  {nm:26s} mean {s[:, i].mean() / 1e3:9.1f} kcyc  max {s[:, i].max() / 1e3:9.1f}")
