#!/bin/bash
# per-stage clock accounting of edge_fused_kernel (thread 0's clock64 between
# the EDGE_T markers, summed over CTAs): prints the cycle shares (GPU box)
set -e
# build here first: JB_BUILD_TAG=clk JB_NVCC_EXTRA=-DEDGE_STAGE_CLOCKS python -m paper_2503_10855_b200.build
cd $GRAFT_REPO_ROOT
python - <<'PY'
import ctypes, numpy as np, torch, sys
NF = 64
sys.path.insert(0, '.')
from paper_2503_10855_b200 import workloads as W
import os; lib = ctypes.CDLL(os.environ.get('CLK_LIB', 'paper_2503_10855_b200/libjunob200_clk.so'))
g, st, sx, sy, th = W.edge_filters()
x = torch.from_numpy(W.edge_batch(NF, 1080, 1920)).cuda()
out = torch.empty_like(x)
f = [torch.from_numpy(a).cuda() for a in (g, st, sx, sy)]
for _ in range(3):
    lib.jb_edge_f32(ctypes.c_uint64(NF), ctypes.c_uint64(1080), ctypes.c_uint64(1920), ctypes.c_uint64(7), ctypes.c_uint64(3), ctypes.c_uint64(3),
                    ctypes.c_void_p(x.data_ptr()), *[ctypes.c_void_p(t.data_ptr()) for t in f], ctypes.c_float(float(th)),
                    ctypes.c_void_p(out.data_ptr()), ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * 16)()
lib.jb_edge_stage_clocks(buf)
v = np.array(list(buf)[:10], dtype=np.float64)
names = ["0 stage0 copy + barrier", "1 gaussian + barrier", "2 laplacian + barrier", "3 zero-cross (generic)", "4 sobel + unit pick + barrier", "5 reject unit", "6 tile top: probes", "7 bulk store + atomicMax issue", "8 tile top: slot wait", "9 count previous tile (flush_done)"]
for n_, c in zip(names, v): print(f"{n_:22s} {c / v.sum() * 100:5.1f}%  {c / 3 / 444 / 1.965e3:9.1f} us/CTA/call")
PY
