#!/bin/bash
# one `ncu --set full` capture of each workload's dominant kernel (1 launch) +
# the launch list of the default bench; reports into gpurun_out/
#   SPECS="srad srad_strip 3;euler euler_rk 3"   (workload kernel-regex skip)
mkdir -p gpurun_out
prof() {  # workload kernel-regex skip
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$2 -s ${3:-2} -c 1 \
     -o gpurun_out/prof_$1 -f python bench.py --workload $1 --steps 1 --warmup 3 --no-cpu --e2e-steps 1 \
     > gpurun_out/ncu_$1.log 2>&1 || echo "ncu $1 failed" >> gpurun_out/ncu_failures.log
}
SPECS=${SPECS:-"edge edge_fused 3;matmul gemm_3xtf32 3;srad srad_ 3;euler euler_rk 3;bfs bfs_kernel 1;backprop bp_adjust 1;cava cava_kernel 1"}
IFS=';' read -ra LIST <<< "$SPECS"
for spec in "${LIST[@]}"; do
  prof $spec
done
if [ -z "${NO_LAUNCHES:-}" ]; then
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_edge.csv \
   python bench.py --steps 2 --warmup 3 --no-cpu --e2e-steps 1 > /dev/null 2>&1
fi
ls gpurun_out/*.ncu-rep
