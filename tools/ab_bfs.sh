#!/bin/bash
# BFS build variants (JB_BUILD_TAG libs): parity + bench each
set -u
OUT=gpurun_out; mkdir -p $OUT
for tag in "" ${TAGS:-}; do
  L=paper_2503_10855_b200/libjunob200${tag:+_$tag}.so
  JB_LIB=$L timeout 300 python -m pytest tests/test_rodinia_gpu.py -x -q -k bfs > $OUT/ab_bfs_t$tag.log 2>&1
  JB_LIB=$L timeout 300 python bench.py --workload bfs --steps 10 --warmup 3 --no-cpu > $OUT/ab_bfs$tag.json 2>/dev/null
  python -c "import json;d=json.load(open('$OUT/ab_bfs$tag.json'));r=d['roofline'];print('bfs[$tag]', d['value'], r['frac'], r['avg_launch_ms'], '$(tail -1 $OUT/ab_bfs_t$tag.log)')"
done
