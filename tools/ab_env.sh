#!/bin/bash
# A/B of an environment variable on the default bench: VAR=name VALUES="a b c" bash tools/ab_env.sh
set -u
for r in 1 2; do for v in ${VALUES}; do
  echo -n "[$VAR=$v] "; env $VAR=$v python bench.py --steps 10 --warmup 3 --no-cpu --e2e-steps 1 ${BENCH_ARGS:-} 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.readline()); print(d['value'], d['roofline']['avg_launch_ms'])"
done; done
