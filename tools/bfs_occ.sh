#!/bin/bash
# BFS occupancy / L1 carveout sweep (JB_BFS_CARVE percent, JB_BFS_CTAS cap)
set -u
mkdir -p gpurun_out
for cfg in "-1 0" "0 0" "10 0" "20 0" "30 0" "30 1" "44 0" "44 1" "100 0"; do
  set -- $cfg
  JB_BFS_VERBOSE=1 JB_BFS_CARVE=$1 JB_BFS_CTAS=$2 timeout 300 python bench.py --workload bfs --steps 10 --warmup 3 --no-cpu > gpurun_out/occ.json 2> gpurun_out/occ.err
  echo "carve=$1 ctas=$2 $(grep -m1 'CTAs/SM' gpurun_out/occ.err) $(python -c "import json;d=json.load(open('gpurun_out/occ.json'));print(d['value'], d['roofline']['avg_launch_ms'])")"
done
