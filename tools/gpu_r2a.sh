#!/bin/bash
# Round-2 first GPU pass: gpu tests, default bench, reference arm, the e2e
# path through api.execute for every workload.
set -u
mkdir -p gpurun_out
OUT=gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/gpu.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 1200 python -m pytest tests -m gpu -x -q ${PYTEST_ARGS:-} > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 600 python bench.py --steps 20 --warmup 5 > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $OUT/bench.err
( time timeout 900 python bench.py --impl reference --steps 20 --warmup 5 ) > $OUT/bench_ref.json 2> $OUT/bench_ref.err
for w in matmul srad euler bfs backprop cava; do
  timeout 600 python bench.py --workload $w --steps 10 --warmup 3 >> $OUT/bench_all.jsonl 2>> $OUT/bench_all.err
done
tail -3 $OUT/smoke.log; tail -5 $OUT/pytest_gpu.log; cat $OUT/bench.json; tail -3 $OUT/bench.err; cat $OUT/bench_ref.json; tail -4 $OUT/bench_ref.err
