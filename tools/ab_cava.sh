#!/bin/bash
# CAVA bench A/B of library variants (P=4096 compute variant and P=16): TAGS="a" bash tools/ab_cava.sh
for r in 1 2; do for tag in "" ${TAGS:-}; do
  L=paper_2503_10855_b200/libjunob200${tag:+_$tag}.so
  echo -n "[$tag] "; JB_LIB=$L python bench.py --workload cava --ctrl-pts 4096 --batch 8 --steps 5 --warmup 3 --no-cpu --e2e-steps 1 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.readline()); print('P4096', d['value'])"
  echo -n "[$tag] "; JB_LIB=$L python bench.py --workload cava --no-cpu --e2e-steps 1 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.readline()); print('P16', d['value'])"
done; done
