for tag in "" pm512 pm1024; do
  L=paper_2503_10855_b200/libjunob200${tag:+_$tag}.so
  for r in 1 2; do
    echo -n "[$tag] "; JB_LIB=$L python bench.py --workload cava --ctrl-pts 4096 --batch 8 --steps 5 --warmup 3 --no-cpu --e2e-steps 1 | python -c "import sys,json; d=json.loads(sys.stdin.readline()); print('P4096', d['value'])"
    echo -n "[$tag] "; JB_LIB=$L python bench.py --workload cava --no-cpu --e2e-steps 1 | python -c "import sys,json; d=json.loads(sys.stdin.readline()); print('P16', d['value'])"
  done
done
