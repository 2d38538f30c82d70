#!/bin/bash
# One iteration on the GPU box: selected gpu tests, bench lines, ncu captures.
#   TESTS="-k srad"  WORKLOADS="srad"  SPECS="srad srad_ 3"
set -u
mkdir -p gpurun_out
OUT=gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q ${TESTS_K:+-k "$TESTS_K"} > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
: > $OUT/bench_iter.jsonl
for w in ${WORKLOADS:-}; do
  timeout 600 python bench.py --workload $w ${BENCH_ARGS:---steps 5 --warmup 3 --no-cpu} >> $OUT/bench_iter.jsonl 2> $OUT/bench_$w.err || echo "{\"workload\": \"$w\", \"failed\": true}" >> $OUT/bench_iter.jsonl
done
if [ -n "${SPECS:-}" ]; then SPECS="$SPECS" bash tools/ncu_all.sh > /dev/null 2>&1; fi
tail -15 $OUT/pytest_gpu.log
python - <<'PY'
import json
for l in open("gpurun_out/bench_iter.jsonl"):
    d = json.loads(l)
    r = d.get("roofline") or {}
    print(d.get("metric"), d.get("value"), d.get("unit"), "| e2e", (d.get("e2e") or {}).get("value"),
          "| roof", r.get("achieved"), r.get("unit"), r.get("frac"), "| launch ms", r.get("avg_launch_ms"), d.get("failed", ""))
PY
for f in $OUT/bench_*.err; do [ -s $f ] && { echo "== $f"; tail -5 $f; }; done
true
