#!/bin/bash
# A/B of library build variants (JB_BUILD_TAG libs) on one workload: parity tests (-k $K) + bench
set -u
for tag in "" ${TAGS:-}; do
  L=paper_2503_10855_b200/libjunob200${tag:+_$tag}.so
  R=$(JB_LIB=$L timeout 600 python -m pytest tests -m gpu -x -q -k "${K}" 2>&1 | tail -1)
  for r in 1 2; do
    echo -n "[$tag] "; JB_LIB=$L python bench.py --workload $W --steps 10 --warmup 3 --no-cpu --e2e-steps 1 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.readline()); print(d['value'], d['roofline']['frac'], '$R')"
  done
done
