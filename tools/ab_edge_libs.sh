#!/bin/bash
# edge bench with library variants: TAGS="a b" bash tools/ab_edge_libs.sh
for r in 1 2; do for tag in "" ${TAGS:-}; do
  L=paper_2503_10855_b200/libjunob200${tag:+_$tag}.so
  echo -n "[$tag] "; JB_LIB=$L python bench.py --steps 10 --warmup 3 --no-cpu --e2e-steps 1 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.readline()); print(d['value'], d['roofline']['avg_launch_ms'])"
done; done
