#!/bin/bash
# Round-2 re-baseline: smoke, gpu tests, default bench + reference arm, every
# workload's bench line, the default bench's ncu launch list.
set -u
mkdir -p gpurun_out; OUT=gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/gpu.txt 2>&1
lscpu > $OUT/lscpu.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 1500 python -m pytest tests -m gpu -q ${PYTEST_ARGS:-} > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 600 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $OUT/bench.err
( time timeout 900 python bench.py --impl reference ) > $OUT/bench_ref.json 2> $OUT/bench_ref.err
rm -f $OUT/bench_all.jsonl
for w in matmul srad euler bfs backprop cava; do
  timeout 600 python bench.py --workload $w --steps 10 --warmup 3 >> $OUT/bench_all.jsonl 2>> $OUT/bench_all.err
done
timeout 600 python bench.py --workload cava --ctrl-pts 4096 --batch 16 --steps 5 --warmup 3 >> $OUT/bench_all.jsonl 2>> $OUT/bench_all.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --e2e-steps 1 > $OUT/ncu_launch.log 2>&1
tail -3 $OUT/smoke.log; tail -15 $OUT/pytest_gpu.log; cat $OUT/bench.json; tail -3 $OUT/bench.err; cat $OUT/bench_ref.json; tail -4 $OUT/bench_ref.err
python - <<'P'
import json
for l in open("gpurun_out/bench_all.jsonl"):
    d=json.loads(l); r=d.get("roofline") or {}
    print(d["config"].get("workload"), d["value"], d["unit"], "frac", r.get("frac"), "avg", r.get("avg_launch_ms"), "e2e", d["e2e"]["value"], "cpu", (d.get("cpu_baseline") or {}).get("value"), d.get("parity_spot_check"))
P
