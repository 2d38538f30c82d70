#!/bin/bash
# matmul pair kernel: tests (bounded), bench both kernels, ncu of the pair kernel
set -u
mkdir -p gpurun_out; OUT=gpurun_out
timeout 300 python -m pytest tests/test_matmul_gpu.py -x -q > $OUT/mm_tests.log 2>&1; echo "rc=$?" >> $OUT/mm_tests.log
tail -5 $OUT/mm_tests.log
for v in 1 0; do
  JB_MM_PAIR=$v timeout 300 python bench.py --workload matmul --steps 20 --warmup 5 --no-cpu > $OUT/mm_bench_$v.json 2> $OUT/mm_bench_$v.err
  python -c "import json;d=json.load(open('$OUT/mm_bench_$v.json'));r=d['roofline'];print('pair=$v', d['value'], r['frac'], r['avg_launch_ms'], d['e2e']['value'], d.get('parity_spot_check'))" || tail -5 $OUT/mm_bench_$v.err
done
timeout 300 ncu --set full --clock-control none --import-source on -k regex:gemm_3xtf32_pair -s 3 -c 1 -o $OUT/prof_mm_pair -f python bench.py --workload matmul --steps 1 --warmup 3 --no-cpu --e2e-steps 1 > $OUT/ncu_mm.log 2>&1
tail -3 $OUT/ncu_mm.log
