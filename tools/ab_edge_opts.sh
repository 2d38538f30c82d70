for r in 1 2; do for v in "" wnm; do for o in 0 1; do
  if [ -n "$v" ]; then export JB_LIB=paper_2503_10855_b200/libjunob200_$v.so; else unset JB_LIB; fi
  echo -n "[$v opts=$o] "; JB_EDGE_OPTS=$o python bench.py --steps 10 --warmup 3 --no-cpu --e2e-steps 1 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.readline()); print(d['value'], d['roofline']['avg_launch_ms'])"
done; done; done
