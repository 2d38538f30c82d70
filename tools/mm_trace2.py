"""Per-CTA phase timeline of the CTA-pair tcgen05 matmul (build: JB_BUILD_TAG=trace
JB_NVCC_EXTRA=-DMM_TRACE python -m paper_2503_10855_b200.build; run with
JB_LIB=paper_2503_10855_b200/libjunob200_trace.so)."""
import ctypes, os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_10855_b200 import _lib, workloads as W
lib = _lib.load()
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
a, b = W.matmul_inputs(n, n, n)
da, db = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
dc = torch.empty((n, n), device="cuda")
flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
for it in range(3):
    flush.fill_(1)
    torch.cuda.synchronize()
    lib.jb_matmul_f32(n, n, n, da.data_ptr(), db.data_ptr(), dc.data_ptr(), torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
buf = np.zeros((512, 12), np.uint64)
lib.jb_mm_trace(ctypes.c_void_p(buf.ctypes.data))
ncta = 128
t = buf[:ncta].astype(np.int64)
t0 = t[:, 0].min()
names = ["start", "setup synced", "first TMA landed", "first MMA", "last MMA issued", "accum ready",
         "partials written", "all splits in", "stores done"]
for i, nm in enumerate(names):
    v = (t[:, i] - t0) / 1e3
    ok = t[:, i] > 0
    if ok.any():
        v = v[ok]
        print(f"{nm:18s} min {v.min():7.2f}  med {np.median(v):7.2f}  max {v.max():7.2f} us  (n={ok.sum()})")
for i, nm in ((10, "MMA waits conv"), (11, "conv waits lo slot")):
    v = buf[:ncta, i].astype(np.float64) / 1e3 / 3  # accumulated over the 3 calls
    v = v[v > 0]
    if len(v):
        print(f"{nm:18s} per CTA: med {np.median(v):7.2f} us total (n={len(v)})")
