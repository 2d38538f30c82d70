set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/bench_edge.json 2> gpurun_out/bench_edge.err
timeout 600 python bench.py --workload matmul --steps 20 --warmup 5 > gpurun_out/bench_mm.json 2> gpurun_out/bench_mm.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_3xtf32 -s 3 -c 1 -o gpurun_out/prof_mm -f python bench.py --workload matmul --steps 2 --warmup 3 --no-cpu --e2e-steps 1 > gpurun_out/ncu_mm.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_mm.csv python bench.py --workload matmul --steps 3 --warmup 3 --no-cpu --e2e-steps 1 > /dev/null 2>&1
tail -15 gpurun_out/pytest_gpu.log; cat gpurun_out/bench_edge.json gpurun_out/bench_mm.json; tail -3 gpurun_out/bench_mm.err gpurun_out/bench_edge.err
