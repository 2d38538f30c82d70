"""Where the edge end-to-end time goes: PCIe H2D alone (registered caller
memory vs torch pinned memory), the pipeline without kernels, and the full
pipelined call at several chunk sizes.  Prints one line per probe."""
import time

import numpy as np
import torch

from paper_2503_10855_b200 import api, hostmem
from paper_2503_10855_b200 import workloads as W

B, n, m = 256, 1080, 1920
x_np = W.edge_batch(B, n, m, seed=1000)
g, st, sx, sy, th = W.edge_filters()
dev = torch.device("cuda", 0)
xr = hostmem.pinned_view(x_np)
xp = torch.from_numpy(x_np).pin_memory()
buf = torch.empty((16, n, m), device=dev)


def h2d(src, chunk=16, reps=3):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        t = time.perf_counter()
        for f0 in range(0, B, chunk):
            buf[:chunk].copy_(src[f0:f0 + chunk], non_blocking=True)
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t)
    return B * n * m * 4 / best / 1e9


print(f"h2d registered caller memory: {h2d(xr):.1f} GB/s")
print(f"h2d torch pinned memory:      {h2d(xp):.1f} GB/s")
for chunk in (8, 16, 32):
    for bits in (True, False):
        out = torch.empty((B, n, m), dtype=torch.float32).pin_memory()
        best = 1e9
        for _ in range(4):
            torch.cuda.synchronize()
            t = time.perf_counter()
            api.edge_detection_pipelined(xr, g, st, sx, sy, th, out=out, chunk=chunk, bits=bits)
            torch.cuda.synchronize()
            best = min(best, time.perf_counter() - t)
        print(f"pipelined chunk={chunk} bits={bits}: {B / best:.0f} frames/s ({best * 1e3:.1f} ms)")
best = 1e9
for _ in range(4):
    t = time.perf_counter()
    api.execute("edge_detection", [n, m, 7, 3, 3], [x_np, g, st, sx, sy, th])
    best = min(best, time.perf_counter() - t)
print(f"api.execute numpy: {B / best:.0f} frames/s ({best * 1e3:.1f} ms)")
