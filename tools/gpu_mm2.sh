#!/bin/bash
set -u
mkdir -p gpurun_out; OUT=gpurun_out
timeout 300 python -m pytest tests/test_matmul_gpu.py tests/test_cli.py -x -q -m gpu > $OUT/mm_tests.log 2>&1; echo "rc=$?" >> $OUT/mm_tests.log
echo "tests: $(tail -2 $OUT/mm_tests.log | tr '\n' ' ')"
JB_MM_BNP=128 timeout 300 python -m pytest tests/test_matmul_gpu.py -x -q -m gpu > $OUT/mm_tests128.log 2>&1; echo "rc=$?" >> $OUT/mm_tests128.log
echo "tests128: $(tail -2 $OUT/mm_tests128.log | tr '\n' ' ')"
for B in 256 128; do
  echo "== trace BNP=$B"; JB_MM_BNP=$B JB_LIB=paper_2503_10855_b200/libjunob200_trace.so timeout 120 python tools/mm_trace2.py
  JB_MM_BNP=$B timeout 300 python bench.py --workload matmul --steps 20 --warmup 5 --no-cpu > $OUT/mm_bench$B.json 2> $OUT/mm_bench$B.err
  python -c "import json;d=json.load(open('$OUT/mm_bench$B.json'));r=d['roofline'];print('BNP=$B', d['value'], r['frac'], r['avg_launch_ms'], d['e2e']['value'])" || tail -5 $OUT/mm_bench$B.err
done
