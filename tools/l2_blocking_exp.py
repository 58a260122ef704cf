"""Experiment: L2-blocked schedule (kb_capi.cu sfista_blocked) vs the whole-plane schedule.

usage: python tools/l2_blocking_exp.py cfg5 [iters] -- times `iters` iterations of the config's
solve for several KB_L2_STRIP / KB_L2_GROUP settings (no graph, so the setting can change per
call) and checks each result against the unblocked one."""

import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1901_00913_b200 as kb  # noqa: E402
from paper_1901_00913_b200 import workloads as W  # noqa: E402
from paper_1901_00913_b200.device import INT_MAX, DeviceOperator, device_operator  # noqa: E402

cfgname = sys.argv[1] if len(sys.argv) > 1 else "cfg5"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 10
cfg = W.CONFIGS[cfgname]
torch.cuda.set_device(0)
t0 = time.time()
if cfg.batch > 1:
    nimg = cfg.batch
    ops, Bs = [], []
    for i in range(nimg):
        _, psf, B = W.make_image_data(cfg, seed=0, index=i, device="cuda")
        ops.append(kb.decompose(psf, kb.BoundaryCondition(cfg.bc), s=cfg.r, shape=(cfg.m, cfg.m)))
        Bs.append(B)
    dev = DeviceOperator(ops, "float32")
    Bd = torch.from_numpy(np.stack(Bs)).to("cuda", torch.float32)
    L = np.full(nimg, 1.0)
    key = "KB_L2_GROUP"
    settings = ["0", "4", "8", "16", "32"]
else:
    X, psf, B = W.make_image_data(cfg, seed=0, device="cuda")
    op = kb.decompose(psf, kb.BoundaryCondition(cfg.bc), s=cfg.r, shape=(cfg.m, cfg.m))
    dev = device_operator(op, "float32")
    Bd = torch.from_numpy(B).to("cuda", torch.float32)
    L = 1.0
    key = "KB_L2_STRIP"
    settings = ["0", "128", "256", "512", "1024"]
print(f"setup {time.time() - t0:.1f} s", flush=True)
_, beta = kb.momentum_table(iters)
flag = torch.full((1,), INT_MAX, dtype=torch.int32, device="cuda")
ref = None
out = {}
for st in settings + ["0"]:
    os.environ[key] = st
    Xd, Yd = torch.zeros_like(Bd), torch.zeros_like(Bd)
    dev.sfista_run(Bd, Xd, Yd, beta, 0, 2, L, cfg.lam, True, flag)  # warm-up
    times = []
    for rep in range(3):
        Xd.zero_(); Yd.zero_()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        dev.sfista_run(Bd, Xd, Yd, beta, 0, iters, L, cfg.lam, True, flag)
        e1.record()
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1) / iters)
    if ref is None:
        ref = Xd.clone()
        diff = 0.0
    else:
        diff = float((Xd - ref).abs().max() / ref.abs().max())
    ms = min(times)
    mpix = cfg.batch * cfg.m * cfg.m / 1e6 / (ms / 1e3)
    print(json.dumps({key: st, "ms_per_iter": round(ms, 4), "mpix_it_s": round(mpix, 1),
                      "max_rel_diff_vs_unblocked": diff}), flush=True)
