#!/bin/bash
# SRAD tolerance-mode iteration: tests, bench of the variants, ncu of the kernel.
set -u
mkdir -p gpurun_out; OUT=gpurun_out
timeout 900 python -m pytest tests/test_rodinia_gpu.py tests/test_property_gpu.py tests/test_dist_gpu.py tests/test_runner.py -x -q -k "srad or runner" > $OUT/srad_tests.log 2>&1; echo "rc=$?" >> $OUT/srad_tests.log
for tag in "" _m2 _m4; do
  JB_LIB=paper_2503_10855_b200/libjunob200$tag.so timeout 300 python bench.py --workload srad --steps 10 --warmup 3 --no-cpu > $OUT/srad_bench$tag.json 2> $OUT/srad_bench$tag.err
done
timeout 900 python -m pytest tests/test_fullsize_gpu.py -x -q -k srad > $OUT/srad_full.log 2>&1; echo "rc=$?" >> $OUT/srad_full.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:srad_strip -s 3 -c 1 -o $OUT/prof_srad_tol -f python bench.py --workload srad --steps 2 --warmup 3 --no-cpu --e2e-steps 1 > $OUT/ncu_srad.log 2>&1
tail -3 $OUT/srad_tests.log; tail -3 $OUT/srad_full.log
for tag in "" _m2 _m4; do python -c "import json;d=json.load(open('$OUT/srad_bench$tag.json'));print('$tag', d['value'], d['roofline']['frac'], d['e2e']['value'])"; done
