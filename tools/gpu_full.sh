#!/bin/bash
# Full GPU round: smoke, gpu tests, every workload's bench line, ncu captures.
set -u
mkdir -p gpurun_out
OUT=gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/gpu.txt 2>&1
lscpu > $OUT/lscpu.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 1200 python -m pytest tests -m gpu -x -q ${PYTEST_ARGS:-} > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
bash tools/bench_all.sh > /dev/null 2>&1
[ -z "${NO_NCU:-}" ] && bash tools/ncu_all.sh > /dev/null 2>&1
tail -3 $OUT/smoke.log; tail -8 $OUT/pytest_gpu.log; cat $OUT/bench_all.jsonl | cut -c1-400
