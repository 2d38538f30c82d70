#!/bin/bash
# One GPU round: smoke, gpu tests, bench, ncu launch list + full capture of the
# dominant kernel.  Run under gpurun from the repo root.
set -u
mkdir -p gpurun_out
OUT=gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/gpu.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 900 python -m pytest tests -m gpu -x -q ${PYTEST_ARGS:-} > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 600 python bench.py ${BENCH_ARGS:-} > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $OUT/bench.err
if [ -n "${NCU_KERNEL:-}" ]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
      python bench.py ${NCU_BENCH_ARGS:---steps 2 --warmup 3 --no-cpu --e2e-steps 1} > $OUT/ncu_launch_bench.log 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:${NCU_KERNEL} -s 2 -c 1 \
      -o $OUT/prof_${NCU_KERNEL} -f python bench.py ${NCU_BENCH_ARGS:---steps 2 --warmup 3 --no-cpu --e2e-steps 1} \
      > $OUT/ncu_full.log 2>&1
fi
tail -3 $OUT/smoke.log; tail -5 $OUT/pytest_gpu.log; cat $OUT/bench.json; tail -3 $OUT/bench.err
