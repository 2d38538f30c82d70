#!/bin/bash
# N>1 code path of bench.py on a one-GPU box: 2 ranks share the GPU (gloo
# control plane; the fused CFD exchange is replaced by the NCCL path there:
# its full-size stage grids cannot co-reside on one GPU, tests/test_dist_gpu.py
# covers it at small sizes).  Checks that every workload runs and prints one JSON line
# per arm; the numbers are not scaling results.
mkdir -p gpurun_out
: > gpurun_out/multi_rank.log
for w in ${WORKLOADS:-edge cava matmul srad euler bfs backprop}; do
  for impl in ours reference; do
    echo "== $w $impl" >> gpurun_out/multi_rank.log
    JB_BENCH_SHARE_GPU=1 JB_SRAD_P2P_GRID=8 JB_EULER_NCCL=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
      --master-addr 127.0.0.1 --master-port 29517 bench.py --workload $w --impl $impl --gpus 2 --steps 2 --warmup 3 \
      --e2e-steps 1 >> gpurun_out/multi_rank.log 2>&1
    echo "rc=$?" >> gpurun_out/multi_rank.log
  done
done
echo "== matmul row blocks vs N=1" >> gpurun_out/multi_rank.log
JB_BENCH_SHARE_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29518 tools/matmul_rowblock_check.py >> gpurun_out/multi_rank.log 2>&1
echo "rc=$?" >> gpurun_out/multi_rank.log
grep -E "^==|^rc=|\"metric\"|unavailable|Error|bit-identical|DIFFERENT" gpurun_out/multi_rank.log | cut -c1-220
