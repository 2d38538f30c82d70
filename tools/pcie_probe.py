"""PCIe ceiling for the e2e numbers: pinned H2D alone, D2H alone and both
directions at once, then the pipelined edge/CAVA host-buffer paths at several
chunk sizes.  usage: python tools/pcie_probe.py"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_10855_b200 import api, workloads as W  # noqa: E402

dev = torch.device("cuda", 0)
N = 1 << 30
h_in = torch.empty(N, dtype=torch.uint8).pin_memory()
h_out = torch.empty(N, dtype=torch.uint8).pin_memory()
d_a = torch.empty(N, dtype=torch.uint8, device=dev)
d_b = torch.empty(N, dtype=torch.uint8, device=dev)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=3):
    fn(); torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / reps


res = {}
res["h2d_gbs"] = N / timed(lambda: d_a.copy_(h_in, non_blocking=True)) / 1e9
res["d2h_gbs"] = N / timed(lambda: h_out.copy_(d_b, non_blocking=True)) / 1e9


def both():
    with torch.cuda.stream(s1):
        d_a.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2):
        h_out.copy_(d_b, non_blocking=True)


t = timed(both)
res["bidir_each_gbs"] = N / t / 1e9
del d_a, d_b, h_in, h_out
torch.cuda.empty_cache()

g, st, sx, sy, th = W.edge_filters()
x = torch.from_numpy(W.edge_batch(256, 1080, 1920, seed=1)).pin_memory()
o = torch.empty_like(x).pin_memory()
for ch in (4, 8, 16, 32):
    tt = timed(lambda: api.edge_detection_pipelined(x, g, st, sx, sy, th, out=o, chunk=ch), reps=3)
    res[f"edge_e2e_fps_chunk{ch}"] = round(256 / tt, 1)
res["edge_pcie_each_gbs_chunk_best"] = round(max(v for k, v in res.items() if k.startswith("edge_e2e")) * x[0].numel() * 4 / 1e9, 1)
del x, o
raw = torch.from_numpy(W.cava_raw(64, 1080, 1920)).pin_memory()
ro = torch.empty_like(raw).pin_memory()
prm = W.cava_params(16)
for ch in (1, 2, 4, 8, 16):
    tt = timed(lambda: api.cava_pipelined(raw, *prm, out=ro, chunk=ch), reps=3)
    res[f"cava_e2e_fps_chunk{ch}"] = round(64 / tt, 1)
print(json.dumps({k: (round(v, 2) if isinstance(v, float) else v) for k, v in res.items()}))
