"""Per-role wait / busy cycles of the fused kernel (needs a -DKB_FU_PROF=1 build; KB_FUSED=1).

usage: fu_profile.py [cfg] [m] [adjoint 0/1]  -- block means of kb_fused.cuh FuProf slots (kcycles)
"""
import ctypes, os, sys, time
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
_, psf, B = W.make_image_data(cfg, seed=0, device="cuda", m=m, counts=(cfg.n_rect, cfg.n_disk) if m == cfg.m else (200, 100))
op = kb.decompose(psf, kb.BoundaryCondition(cfg.bc), s=cfg.r, shape=(m, m))
dev = device_operator(op, "float32")
print("info", dev.info(), "bands", dev.bands, flush=True)
Bd = torch.from_numpy(B).to("cuda", torch.float32)
out = torch.empty_like(Bd)
for _ in range(3):
    dev.apply(Bd, out=out, adjoint=adj)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
reps = 20
e0.record()
for _ in range(reps):
    dev.apply(Bd, out=out, adjoint=adj)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
buf = (ctypes.c_ulonglong * (2 * 1024 * 8))()
assert load_library().kb_debug_trace(buf, 2 * 1024 * 8) == 0
a = np.frombuffer(buf, dtype=np.uint64).reshape(2, 1024, 8).astype(np.float64)
slots = np.concatenate([a[0], a[1]], axis=1)  # [block][16]
slots = slots[slots[:, 11] > 0]
names = ["A-issuer a_ready wait", "A-issuer acc/brick wait", "B-issuer b_ready wait", "B-issuer acc/brick wait",
         "Xconv a_free wait", "Xconv xfull wait", "drain accA_full wait", "Zconv b_free wait",
         "drain ld+sts", "drain bar waits", "epi accB_full wait", "Xconv total", "Xconv busy", "Zconv busy",
         "epi busy", "producer waits"]
print(f"{name} m={m} adj={adj}: {ms:.3f} ms per application (events, 20 reps), {len(slots)} blocks")
if not len(slots):
    sys.exit(0)  # not a -DKB_FU_PROF=1 build
for i, nm in enumerate(names):
    print(f"  {i:2d} {nm:26s} mean {slots[:, i].mean() / 1e3:10.1f} kcyc  max {slots[:, i].max() / 1e3:10.1f}")
