"""Event timeline of block 0 of the fused kernel (needs a -DKB_FU_TRACE=1 build; KB_FUSED=1).

usage: fu_timeline.py [cfg] [m] [adjoint]  -- per term: event times (kcycles from the first event)
"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1901_00913_b200 as kb
from paper_1901_00913_b200 import workloads as W
from paper_1901_00913_b200.device import device_operator, load_library
name = sys.argv[1] if len(sys.argv) > 1 else "cfg5"
cfg = W.CONFIGS[name]
m = int(sys.argv[2]) if len(sys.argv) > 2 else 2048
adj = bool(int(sys.argv[3])) if len(sys.argv) > 3 else False
_, psf, B = W.make_image_data(cfg, seed=0, device="cuda", m=m, counts=(200, 100))
op = kb.decompose(psf, kb.BoundaryCondition(cfg.bc), s=cfg.r, shape=(m, m))
dev = device_operator(op, "float32")
Bd = torch.from_numpy(B).to("cuda", torch.float32)
for _ in range(2):
    dev.apply(Bd, adjoint=adj)
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * (2 * 1024 * 8))()
assert load_library().kb_debug_trace(buf, 2 * 1024 * 8) == 0
a = np.frombuffer(buf, dtype=np.uint64).astype(np.float64).reshape(16, 1024)[:9]
n = int((a[0] > 0).sum())
t0 = a[:, :n][a[:, :n] > 0].min()
names = ["A start", "A commit", "drain got", "drain done", "Zconv done", "B first", "B commit", "X first", "X last"]
print("term " + " ".join(f"{x:>10s}" for x in names))
for u in range(min(n, 60)):
    print(f"{u:4d} " + " ".join(f"{(a[i, u] - t0) / 1e3:10.2f}" for i in range(9)))
d = np.diff(a[1, :n])
print("A commit interval: mean %.2f kcyc" % (d[d > 0].mean() / 1e3))
flat = np.frombuffer(buf, dtype=np.uint64).astype(np.float64)
st = flat[9216:9216 + 8 * 512].reshape(8, 32, 16)
snames = ["X stored", "A got", "A commit", "Z stored", "B got", "B commit", "B 1st mma", "B last mma"]
for u in (20, 21, 22):
    print(f"term {u} per-stage (kcyc from t0):")
    for i, nm in enumerate(snames):
        row = st[i, u]
        print(f"  {nm:9s} " + " ".join(f"{(x - t0) / 1e3:7.2f}" if x > 0 else "      -" for x in row))
