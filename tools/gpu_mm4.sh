#!/bin/bash
set -u
mkdir -p gpurun_out; OUT=gpurun_out
for L in "" _a1smem; do
JB_MM_PAIR=0 JB_LIB=paper_2503_10855_b200/libjunob200$L.so timeout 300 python -m pytest tests/test_matmul_gpu.py -x -q -m gpu > $OUT/mm_tests$L.log 2>&1; echo "rc=$?" >> $OUT/mm_tests$L.log
echo "tests$L: $(tail -2 $OUT/mm_tests$L.log | tr '\n' ' ')"
for v in 0 1; do
JB_MM_PAIR=$v JB_LIB=paper_2503_10855_b200/libjunob200$L.so timeout 300 python bench.py --workload matmul --steps 30 --warmup 5 --no-cpu > $OUT/mm_bench$v$L.json 2> $OUT/mm_bench$v$L.err
python -c "import json;d=json.load(open('$OUT/mm_bench$v$L.json'));r=d['roofline'];print('lib$L pair=$v', d['value'], r['frac'], r['avg_launch_ms'])" || tail -5 $OUT/mm_bench$v$L.err
done
done
JB_MM_PAIR=0 timeout 300 ncu --metrics gpu__time_duration.sum,sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:gemm -c 3 --csv python bench.py --workload matmul --steps 3 --warmup 3 --no-cpu --e2e-steps 1 2>/dev/null | grep gemm | cut -d, -f5,15,16 | tail -4
