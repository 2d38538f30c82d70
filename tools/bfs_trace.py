"""Per-level timeline of the BFS kernel (build: JB_BUILD_TAG=trace
JB_NVCC_EXTRA='-DMM_TRACE -DBFS_TRACE' python -m paper_2503_10855_b200.build;
run with JB_LIB=paper_2503_10855_b200/libjunob200_trace.so)."""
import ctypes, os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_10855_b200 import _lib, workloads as W
lib = _lib.load()
st, deg, ed = W.bfs_graph()
n, m = len(st), len(ed)
d = [torch.from_numpy(x.view(np.int32)).cuda() for x in (st, deg, ed)]
cost = torch.empty(n, dtype=torch.int32, device="cuda")
s = torch.cuda.current_stream().cuda_stream
for _ in range(3):
    lib.jb_bfs(n, m, d[0].data_ptr(), d[1].data_ptr(), d[2].data_ptr(), 0, cost.data_ptr(), s)
torch.cuda.synchronize()
buf = np.zeros(64, np.uint64)
lib.jb_bfs_trace(ctypes.c_void_p(buf.ctypes.data))
t = buf.astype(np.int64)
nz = np.nonzero(t)[0]
last = nz.max()
sizes = np.bincount(cost.cpu().numpy()[cost.cpu().numpy() >= 0])
for i in range(last):
    f = sizes[i] if i < len(sizes) else 0
    print(f"level {i:2d}: {(t[i + 1] - t[i]) / 1e3:8.2f} us  frontier {f:9d}")
print(f"total to last level start: {(t[last] - t[0]) / 1e3:.1f} us")
