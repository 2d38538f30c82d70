#!/bin/bash
# BFS: parity tests, per-level trace, bench line
set -u
mkdir -p gpurun_out; OUT=gpurun_out
timeout 600 python -m pytest tests -x -q -m gpu -k "bfs" > $OUT/bfs_tests.log 2>&1; echo "rc=$?" >> $OUT/bfs_tests.log
echo "tests: $(tail -2 $OUT/bfs_tests.log | tr '\n' ' ')"
JB_LIB=paper_2503_10855_b200/libjunob200_trace.so timeout 120 python tools/bfs_trace.py
timeout 300 python bench.py --workload bfs --steps 10 --warmup 3 --no-cpu > $OUT/bfs_bench.json 2> $OUT/bfs_bench.err
python -c "import json;d=json.load(open('$OUT/bfs_bench.json'));r=d['roofline'];print('bfs', d['value'], r['frac'], r['avg_launch_ms'], d['e2e']['value'], d.get('parity_spot_check'))" || tail -5 $OUT/bfs_bench.err
