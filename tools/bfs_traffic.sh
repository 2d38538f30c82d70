#!/bin/bash
# BFS build variants (TAGS): bench + ncu DRAM traffic of bfs_kernel
set -u
mkdir -p gpurun_out
for tag in "" ${TAGS:-}; do
  L=paper_2503_10855_b200/libjunob200${tag:+_$tag}.so
  JB_BFS_VERBOSE=1 JB_LIB=$L timeout 300 python bench.py --workload bfs --steps 10 --warmup 3 --no-cpu > gpurun_out/tr.json 2>gpurun_out/tr.err
  v=$(python -c "import json;d=json.load(open('gpurun_out/tr.json'));print(d['value'], d['roofline']['avg_launch_ms'])")
  JB_LIB=$L timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,l1tex__t_sector_hit_rate.pct --clock-control none -k regex:bfs_kernel -c 1 python bench.py --workload bfs --steps 1 --warmup 1 --no-cpu > gpurun_out/tr_ncu$tag.txt 2>&1
  echo "bfs[$tag] $(grep -m1 CTAs gpurun_out/tr.err) $v $(grep -E 'dram__|lts__t_sector_hit|l1tex__t_sector_hit' gpurun_out/tr_ncu$tag.txt | awk '{print $1"="$3$2}' | tr '\n' ' ')"
done
