"""Host<->device staging cost of the public API at cfg5 size (run on the GPU box):
upload_pieces (fp64 host -> fp32 device through pinned pieces) and download_pieces (fp32 device ->
fp64 host), for a few worker counts and piece sizes. python tools/copy_bench.py [m]"""
import sys
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1901_00913_b200 import device as D  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
rng = np.random.default_rng(0)
B = rng.random((m, m))
dst = torch.empty((m, m), dtype=torch.float32, device="cuda")
stage = torch.empty((m, m), dtype=torch.float32, pin_memory=True)
print("cpus", __import__("os").cpu_count())
for workers in (8, 16, 32):
    for piece_mb in (1, 4, 16):
        D._copy_pool = ThreadPoolExecutor(max_workers=workers)
        D._PIECE_BYTES = piece_mb << 20
        up, down, alloc = [], [], []
        for rep in range(4):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            D.upload_pieces(dst, B, stage)
            torch.cuda.synchronize()
            t1 = time.perf_counter()
            out = np.empty((m, m))
            t2 = time.perf_counter()
            D.download_pieces(dst, stage, out)
            torch.cuda.synchronize()
            t3 = time.perf_counter()
            up.append(t1 - t0)
            alloc.append(t2 - t1)
            down.append(t3 - t2)
            del out
        print(f"workers {workers:2d} piece {piece_mb:2d} MiB: upload {min(up) * 1e3:7.1f} ms  download {min(down) * 1e3:7.1f} ms"
              f"  (np.empty {min(alloc) * 1e3:.2f} ms)")
# raw DMA for reference
torch.cuda.synchronize()
t0 = time.perf_counter()
dst.copy_(stage, non_blocking=True)
torch.cuda.synchronize()
t1 = time.perf_counter()
stage.copy_(dst, non_blocking=True)
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"raw pinned DMA of {stage.numel() * 4 / 2**30:.2f} GiB: h2d {(t1 - t0) * 1e3:.1f} ms, d2h {(t2 - t1) * 1e3:.1f} ms")
t0 = time.perf_counter()
s32 = B.astype(np.float32)
t1 = time.perf_counter()
print(f"single-thread astype fp64->fp32: {(t1 - t0) * 1e3:.1f} ms")
