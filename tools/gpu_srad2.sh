#!/bin/bash
set -u
mkdir -p gpurun_out; OUT=gpurun_out
timeout 900 python -m pytest tests/test_rodinia_gpu.py -q -k "srad" > $OUT/srad2_tests.log 2>&1; echo "rc=$?" >> $OUT/srad2_tests.log
for tag in "" _m2 _m4; do
  JB_LIB=paper_2503_10855_b200/libjunob200$tag.so timeout 300 python bench.py --workload srad --steps 3 --warmup 3 --no-cpu --e2e-steps 1 > $OUT/srad_bench$tag.json 2> $OUT/srad_bench$tag.err
done
timeout 900 python -m pytest tests/test_fullsize_gpu.py -q -k "srad_16384_100" > $OUT/srad2_full.log 2>&1; echo "rc=$?" >> $OUT/srad2_full.log
tail -2 $OUT/srad2_tests.log; tail -2 $OUT/srad2_full.log
for tag in "" _m2 _m4; do python -c "import json;d=json.load(open('$OUT/srad_bench$tag.json'));print('srad$tag', d['value'], d['roofline']['frac'], d['roofline']['avg_launch_ms'], d['e2e']['value'], d['clocks'])"; done
