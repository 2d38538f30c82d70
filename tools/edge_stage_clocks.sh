#!/bin/bash
# builds a profiling variant of libjunob200 with per-stage clock accounting of
# edge_fused_kernel and prints the cycle shares (GPU box)
set -e
mkdir -p /tmp/esc && cd /tmp/esc
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -fmad=false -DEDGE_STAGE_CLOCKS -Xcompiler -fPIC \
  -I$GRAFT_REPO_ROOT/include -c $GRAFT_REPO_ROOT/paper_2503_10855_b200/csrc/edge.cu -o edge.o
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -fmad=false -Xcompiler -fPIC \
  -I$GRAFT_REPO_ROOT/include -c $GRAFT_REPO_ROOT/paper_2503_10855_b200/csrc/runtime.cu -o runtime.o
nvcc -gencode arch=compute_100a,code=sm_100a -shared --cudart static -o libedgeclk.so edge.o runtime.o
cd $GRAFT_REPO_ROOT
python - <<'PY'
import ctypes, numpy as np, torch, sys
sys.path.insert(0, '.')
from paper_2503_10855_b200 import workloads as W
lib = ctypes.CDLL('/tmp/esc/libedgeclk.so')
g, st, sx, sy, th = W.edge_filters()
x = torch.from_numpy(W.edge_batch(16, 1080, 1920)).cuda()
out = torch.empty_like(x)
f = [torch.from_numpy(a).cuda() for a in (g, st, sx, sy)]
for _ in range(3):
    lib.jb_edge_f32(ctypes.c_uint64(16), ctypes.c_uint64(1080), ctypes.c_uint64(1920), ctypes.c_uint64(7), ctypes.c_uint64(3), ctypes.c_uint64(3),
                    ctypes.c_void_p(x.data_ptr()), *[ctypes.c_void_p(t.data_ptr()) for t in f], ctypes.c_float(float(th)),
                    ctypes.c_void_p(out.data_ptr()), ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * 8)()
lib.jb_edge_stage_clocks(buf)
v = np.array(list(buf)[:8], dtype=np.float64)
names = ["stage0 load+guard", "gaussian", "laplacian", "zero-cross", "sobel+store+max", "reject help", "slot wait", "done+publish"]
for n_, c in zip(names, v): print(f"{n_:22s} {c / v.sum() * 100:5.1f}%  {c / 3 / 444 / 1.9e3:9.1f} us/CTA/call")
PY
