"""Experiment: cfg5 pass times with the axis roles swapped (the wide 57-tap band first): the
operator of the transposed image, Y^T = sum_i K_i X^T H_i^T (kb_time_passes on both)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1901_00913_b200 as kb
from paper_1901_00913_b200 import workloads as W
from paper_1901_00913_b200.device import DeviceOperator
cfg = W.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg5"]
X, psf, B = W.make_image_data(cfg, seed=0, device="cuda")
op = kb.decompose(psf, kb.BoundaryCondition(cfg.bc), s=cfg.r, shape=(cfg.m, cfg.m))
sw = kb.KronOperator(terms=tuple(kb.KronTerm(sigma=t.sigma, H=t.K, K=t.H) for t in op.terms), shape=op.shape,
                     bc=op.bc, sigma=op.sigma, s=op.s, rank=op.rank, eps=op.eps)
Bd = torch.from_numpy(B).to("cuda", torch.float32)
for name, o in (("as is", op), ("swapped", sw), ("as is", op), ("swapped", sw)):
    dev = DeviceOperator([o], "float32")
    ms = dev.time_passes(Bd, Bd, 1.0, cfg.lam, reps=10)
    print(name, dev.bands, [round(x, 3) for x in ms], round(sum(ms), 3), dev.last_engines(), flush=True)
    del dev
    torch.cuda.empty_cache()
