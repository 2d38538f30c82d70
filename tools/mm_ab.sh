#!/bin/bash
# matmul bench A/B of library variants: TAGS="a b" bash tools/mm_ab.sh
for i in 1 2; do for t in "" ${TAGS:-}; do L=paper_2503_10855_b200/libjunob200${t:+_$t}.so; echo "[$t] $(JB_LIB=$L python bench.py --workload matmul --steps 50 --warmup 5 --no-cpu --e2e-steps 1 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.readline()); print(d['value'], d['roofline']['avg_launch_ms'], d['roofline']['frac'], d['gpu_launches'])")"; done; done
