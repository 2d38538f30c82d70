#!/bin/bash
# edge GPU tests + 2 default bench runs (value, e2e); optional ncu capture (NCU=1)
set -u
mkdir -p gpurun_out
OUT=gpurun_out
timeout 900 python -m pytest tests/test_edge_gpu.py tests/test_fullsize_gpu.py -x -q -k "edge" > $OUT/pytest_edge.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_edge.log
tail -3 $OUT/pytest_edge.log
for i in 1 2; do timeout 600 python bench.py --no-cpu ${BENCH_ARGS:-} > $OUT/bench_q_$i.json 2> $OUT/bench_q_$i.err; done
python - <<'PY'
import json
for i in (1, 2):
    try:
        d = json.loads(open(f"gpurun_out/bench_q_{i}.json").readline())
        print(d["value"], d["e2e"]["value"], d["roofline"]["avg_launch_ms"], d["clocks"])
    except Exception as e:
        print("bench failed", e, open(f"gpurun_out/bench_q_{i}.err").read()[-2000:])
PY
if [ "${NCU:-0}" = 1 ]; then K=edge_fused TAG=${TAG:-edge} bash tools/ncu_src.sh; fi
