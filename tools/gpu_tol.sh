#!/bin/bash
# tolerance-mode SRAD + CFD: tests, benches of build variants, ncu of both kernels.
set -u
mkdir -p gpurun_out; OUT=gpurun_out
timeout 1200 python -m pytest tests/test_rodinia_gpu.py tests/test_property_gpu.py tests/test_dist_gpu.py tests/test_runner.py -q -k "srad or runner or euler" > $OUT/tol_tests.log 2>&1; echo "rc=$?" >> $OUT/tol_tests.log
for tag in "" _m2 _m4; do
  JB_LIB=paper_2503_10855_b200/libjunob200$tag.so timeout 300 python bench.py --workload srad --steps 3 --warmup 3 --no-cpu --e2e-steps 1 > $OUT/srad_bench$tag.json 2> $OUT/srad_bench$tag.err
  JB_LIB=paper_2503_10855_b200/libjunob200$tag.so timeout 300 python bench.py --workload euler --steps 10 --warmup 3 --no-cpu --e2e-steps 1 > $OUT/euler_bench$tag.json 2> $OUT/euler_bench$tag.err
done
timeout 1200 python -m pytest tests/test_fullsize_gpu.py -q -k "srad or euler" > $OUT/tol_full.log 2>&1; echo "rc=$?" >> $OUT/tol_full.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:srad_strip -s 5 -c 1 -o $OUT/prof_srad_tol -f python bench.py --workload srad --steps 1 --warmup 3 --no-cpu --e2e-steps 1 > $OUT/ncu_srad.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:euler_rk -s 6 -c 1 -o $OUT/prof_euler_tol -f python bench.py --workload euler --steps 1 --warmup 3 --no-cpu --e2e-steps 1 > $OUT/ncu_euler.log 2>&1
tail -3 $OUT/tol_tests.log; tail -3 $OUT/tol_full.log
for tag in "" _m2 _m4; do for w in srad euler; do python -c "import json;d=json.load(open('$OUT/${w}_bench$tag.json'));print('$w$tag', d['value'], d['roofline']['frac'], d['roofline']['avg_launch_ms'], d['e2e']['value'])"; done; done
