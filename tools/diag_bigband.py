import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_1901_00913_b200 as kb
from paper_1901_00913_b200 import workloads as W
from paper_1901_00913_b200.device import DeviceOperator
from oracle import kronblur_port as port
for name in ("cfg4", "cfg5"):
    cfg = W.CONFIGS[name]
    for m in (512, 2048):
        psf = W.make_psf(cfg)
        op = kb.decompose(psf, kb.BoundaryCondition(cfg.bc), s=cfg.r, shape=(m, m))
        g = torch.Generator(device="cuda").manual_seed(7)
        X = torch.rand((m, m), generator=g, device="cuda", dtype=torch.float64)
        d64 = DeviceOperator([op], "float64"); AX = d64.apply(X); ATX = d64.apply(X, adjoint=True)
        d32 = DeviceOperator([op], "float32")
        for adj, ref in ((False, AX), (True, ATX)):
            got = d32.apply(X.float(), adjoint=adj).double()
            err = float(torch.linalg.norm(got - ref) / torch.linalg.norm(ref))
            mx = float((got - ref).abs().max() / ref.abs().max())
            print(name, m, "adj" if adj else "fwd", "fp32 vs fp64 rel", err, "max", mx, flush=True)
        if m == 512:
            pop = port.PortOperator(op)
            Xn = X.cpu().numpy()
            print(name, m, "fp64 vs oracle", float(np.linalg.norm(AX.cpu().numpy() - port.kron_apply(pop, Xn)) / np.linalg.norm(port.kron_apply(pop, Xn))))
