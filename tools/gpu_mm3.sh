#!/bin/bash
set -u
mkdir -p gpurun_out; OUT=gpurun_out
timeout 300 python -m pytest tests/test_matmul_gpu.py -x -q -m gpu > $OUT/mm_tests.log 2>&1; echo "rc=$?" >> $OUT/mm_tests.log
echo "tests: $(tail -2 $OUT/mm_tests.log | tr '\n' ' ')"
JB_LIB=paper_2503_10855_b200/libjunob200_trace.so timeout 120 python tools/mm_trace2.py
for v in 1 0; do
JB_MM_PAIR=$v timeout 300 python bench.py --workload matmul --steps 30 --warmup 5 --no-cpu > $OUT/mm_bench$v.json 2> $OUT/mm_bench$v.err
python -c "import json;d=json.load(open('$OUT/mm_bench$v.json'));r=d['roofline'];print('pair=$v', d['value'], r['frac'], r['avg_launch_ms'], d['e2e']['value'])" || tail -5 $OUT/mm_bench$v.err
done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:gemm -c 5 --csv python bench.py --workload matmul --steps 3 --warmup 3 --no-cpu --e2e-steps 1 2>/dev/null | grep gemm | tail -3
