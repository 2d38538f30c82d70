#!/bin/bash
# matmul: GPU tests, per-CTA phase trace, bench line, kernel-only ncu times
set -u
mkdir -p gpurun_out; OUT=gpurun_out
timeout 300 python -m pytest tests/test_matmul_gpu.py tests/test_cli.py -x -q -m gpu > $OUT/mm_tests.log 2>&1; echo "rc=$?" >> $OUT/mm_tests.log
echo "tests: $(tail -2 $OUT/mm_tests.log | tr '\n' ' ')"
JB_LIB=paper_2503_10855_b200/libjunob200_trace.so timeout 120 python tools/mm_trace.py
timeout 300 python bench.py --workload matmul --steps 30 --warmup 5 --no-cpu > $OUT/mm_bench.json 2> $OUT/mm_bench.err
python -c "import json;d=json.load(open('$OUT/mm_bench.json'));r=d['roofline'];print('matmul', d['value'], r['frac'], r['avg_launch_ms'], d['e2e']['value'])" || tail -5 $OUT/mm_bench.err
timeout 300 ncu --metrics gpu__time_duration.sum,sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:gemm -c 3 --csv python bench.py --workload matmul --steps 3 --warmup 3 --no-cpu --e2e-steps 1 2>/dev/null | grep gemm | awk -F'","' '{print $(NF-2), $NF}' | tail -6
