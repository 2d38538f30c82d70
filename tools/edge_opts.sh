#!/bin/bash
# edge in-kernel reject experiments: bench line per JB_EDGE_OPTS value
mkdir -p gpurun_out
for o in ${OPTS:-0 1 2 3}; do
  echo "== opts $o"
  JB_EDGE_OPTS=$o timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu --e2e-steps 1 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l); print(d['value'], d['roofline']['avg_launch_ms'])
    except Exception: print(l.strip()[:300])"
done
echo "== clocks"
JB_EDGE_OPTS=4 timeout 300 python bench.py --steps 1 --warmup 3 --no-cpu --e2e-steps 1 2>&1 | grep "edge clk" | tail -3
