# A/B of library variants on one workload: WL=euler VARIANTS="base" bash tools/ab_workload.sh
for r in 1 2; do for v in "" ${VARIANTS}; do
  if [ -n "$v" ]; then export JB_LIB=paper_2503_10855_b200/libjunob200_$v.so; else unset JB_LIB; fi
  echo -n "[$v] "; python bench.py --workload ${WL:-edge} --steps 5 --warmup 3 --no-cpu --e2e-steps 1 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.readline()); print(d['value'], d['roofline']['avg_launch_ms'])"
done; done
