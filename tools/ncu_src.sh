#!/bin/bash
# One ncu --set full capture with source-line attribution of kernel $K
# (regex) under bench.py $ARGS; writes gpurun_out/src_$TAG.ncu-rep.
set -u
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:${K} -s ${SKIP:-2} -c 1 \
  -o gpurun_out/src_${TAG} -f python bench.py ${ARGS:---steps 2 --warmup 3 --no-cpu --e2e-steps 1} \
  > gpurun_out/src_${TAG}.log 2>&1
echo "ncu rc=$?"; tail -3 gpurun_out/src_${TAG}.log
