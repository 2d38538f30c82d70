"""Row-block matmul across ranks vs the single-device call (bit-identity).

    python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 \
        tools/matmul_rowblock_check.py        (JB_BENCH_SHARE_GPU=1: gloo, one GPU)

Every rank computes its row block of C = A @ B with B broadcast once
(dist.MatmulRowBlocks), C is all-gathered, and rank 0 compares it bit for
bit with jb_matmul_f32 on the whole matrix."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_10855_b200 import api, dist as D, workloads as W  # noqa: E402

share = os.environ.get("JB_BENCH_SHARE_GPU") == "1"
dist.init_process_group("gloo" if share else "nccl")
rank, world = dist.get_rank(), dist.get_world_size()
torch.cuda.set_device(0 if share else int(os.environ.get("LOCAL_RANK", "0")))
n = m = l = 1024
a, b = W.matmul_inputs(n, m, l)
db = torch.from_numpy(b).cuda() if rank == 0 else torch.zeros((m, l), dtype=torch.float32, device="cuda")
mb = D.MatmulRowBlocks(db, n)
c_rows = mb(torch.from_numpy(np.ascontiguousarray(mb.own_rows(a))).cuda())
full = mb.gather(c_rows).cpu().numpy()
if rank == 0:
    ref = api.matmul(a, b)
    same = np.array_equal(full.view(np.uint32), ref.view(np.uint32))
    print(f"matmul row blocks N={world}: {'bit-identical' if same else 'DIFFERENT'} to N=1 "
          f"(max |d| {np.abs(full - ref).max():.3g}), B broadcasts: {mb.broadcasts}", flush=True)
    rc = 0 if same else 1
else:
    rc = 0
dist.barrier()
dist.destroy_process_group()
sys.exit(rc)
