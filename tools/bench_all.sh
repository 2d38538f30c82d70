#!/bin/bash
# every workload once (1 GPU); JSON lines into gpurun_out/bench_all.jsonl
mkdir -p gpurun_out
: > gpurun_out/bench_all.jsonl
for w in ${WORKLOADS:-edge matmul srad euler bfs backprop cava}; do
  timeout 900 python bench.py --workload $w ${BENCH_ARGS:---steps 5 --warmup 3} >> gpurun_out/bench_all.jsonl 2> gpurun_out/bench_$w.err || echo "{\"workload\": \"$w\", \"failed\": true}" >> gpurun_out/bench_all.jsonl
done
cat gpurun_out/bench_all.jsonl
