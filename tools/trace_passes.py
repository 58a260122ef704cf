"""Per-block timeline of the fp64 pass kernels (KB_DEBUG_MODE bit 7, kb_debug_trace).

usage: KB_DEBUG_MODE=128 python tools/trace_passes.py [m] [float64|float32]
(from a -DKB_TRACE=1 build: tools/variant.sh trace -DKB_TRACE=1, run in tmp_variants/trace)
Runs kb_apply (forward: split + plain sum) and one sFISTA iteration (last kernels: adjoint split
+ update sum) on cfg2 and prints, per kernel, the distribution over blocks of each stamp
relative to the kernel's earliest start (us).
split slots: 0 entry, 1 barriers ready, 2 taps loaded, 3 first tile landed, 4 chunk 0 done,
             5 chunk 1 done, 6 exit;  sum slots: 0..3 same, 4 MMA of chunk 0 done,
             5 epilogue of chunk 0 done, 6 exit.
"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1901_00913_b200 as kb
from paper_1901_00913_b200 import workloads as W
from paper_1901_00913_b200.device import device_operator, load_library
from paper_1901_00913_b200.solvers import momentum_table

m = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
dtype = sys.argv[2] if len(sys.argv) > 2 else "float64"
cfg = W.CONFIGS["cfg2"]
_, psf, B = W.make_image_data(cfg, seed=0, m=m, counts=(cfg.n_rect, cfg.n_disk) if m == cfg.m else (50, 25))
op = kb.decompose(psf, kb.BoundaryCondition(cfg.bc), s=cfg.r, shape=(m, m))
dev = device_operator(op, dtype)
Bd = torch.from_numpy(B).to("cuda", dev.tdtype)


def trace():
    torch.cuda.synchronize()
    buf = (ctypes.c_ulonglong * (2 * 1024 * 8))()
    assert load_library().kb_debug_trace(buf, 2 * 1024 * 8) == 0
    return np.frombuffer(buf, dtype=np.uint64).reshape(2, 1024, 8).astype(np.int64)


def report(name, t, kind):
    a = t[kind]
    used = a[:, 0] > 0
    a = a[used]
    t0 = a[:, 0].min()
    print(f"{name}: {used.sum()} blocks, kernel span {(a[:, 6].max() - t0) / 1e3:.2f} us")
    for s in range(7):
        v = a[:, s]
        ok = v > 0
        if not ok.any():
            continue
        r = (v[ok] - t0) / 1e3
        print(f"  slot {s}: min {r.min():7.2f}  p50 {np.median(r):7.2f}  max {r.max():7.2f}  (n={ok.sum()})")
    sm = a[:, 7]
    print(f"  distinct SMs {len(np.unique(sm))}, blocks/SM max {np.bincount(sm).max()}")


for _ in range(3):
    dev.apply(Bd)
t = trace()
report("forward split", t, 0)
report("forward sum (plain)", t, 1)
Xd, Yd = torch.zeros_like(Bd), torch.zeros_like(Bd)
flag = torch.full((1,), 2**31 - 1, dtype=torch.int32, device="cuda")
_, beta = momentum_table(4)
for _ in range(2):
    dev.sfista_run(Bd, Xd, Yd, beta, 0, 1, 1.0, cfg.lam, True, flag, use_graph=False)
t = trace()
report("adjoint split", t, 0)
report("update sum", t, 1)


def by_block(name, t, kind, parts):
    a = t[kind]
    used = a[:, 0] > 0
    n = int(used.sum())
    a = a[:n]
    t0 = a[:, 0].min()
    end = (a[:, 6] - t0) / 1e3
    mma = (a[:, 4] - a[:, 3]) / 1e3
    sm = a[:, 7]
    print(f"{name}: per part index (block = item, part = block % {parts}) mean end / mean stamp4-3")
    for p in range(parts):
        idx = np.arange(n)[np.arange(n) % parts == p]
        print(f"  part {p}: end {end[idx].mean():6.2f} (max {end[idx].max():6.2f})  s4-s3 {mma[idx].mean():6.2f}")
    cnt = np.bincount(sm, minlength=148)
    solo = np.isin(sm, np.nonzero(cnt == 1)[0])
    print(f"  solo-SM blocks: {solo.sum()}, mean end {end[solo].mean() if solo.any() else 0:.2f}; paired mean end {end[~solo].mean():.2f}")
    # partner analysis: for each SM with 2 blocks, end times of both
    slow = np.argsort(end)[-12:]
    print("  slowest blocks (blk, lt, part, sm, end):", [(int(b), int(b) // parts, int(b) % parts, int(sm[b]), round(float(end[b]), 1)) for b in slow])
    fast = np.argsort(end)[:8]
    print("  fastest blocks:", [(int(b), int(b) // parts, int(b) % parts, int(sm[b]), round(float(end[b]), 1)) for b in fast])


by_block("update sum", t, 1, 9)


def by_sm(name, t, kind):
    a = t[kind]
    used = a[:, 0] > 0
    a = a[: int(used.sum())]
    t0 = a[:, 0].min()
    end = (a[:, 6] - t0) / 1e3
    first = (a[:, 3] - t0) / 1e3
    sm = a[:, 7]
    ends = np.zeros(148)
    nb = np.bincount(sm, minlength=148)
    for s_ in range(148):
        if nb[s_]:
            ends[s_] = end[sm == s_].max()
    order = np.argsort(ends)
    print(f"{name}: SM end times (us) p0 {ends[order[0]]:.1f} p10 {np.percentile(ends, 10):.1f} p50 "
          f"{np.median(ends):.1f} p90 {np.percentile(ends, 90):.1f} max {ends.max():.1f}")
    print("  SM id vs end (sorted by id, 8 per row):")
    for r0 in range(0, 148, 16):
        print("   ", " ".join(f"{ends[i]:5.1f}" for i in range(r0, min(r0 + 16, 148))))


by_sm("update sum", t, 1)
by_sm("adjoint split", t, 0)
