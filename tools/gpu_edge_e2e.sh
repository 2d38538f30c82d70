#!/bin/bash
# edge tests + default bench (e2e through the bit-packed D2H) + pcie/expand probe
set -u
mkdir -p gpurun_out
OUT=gpurun_out
timeout 900 python -m pytest tests/test_edge_gpu.py tests/test_abi.py -x -q > $OUT/pytest_edge.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_edge.log
tail -3 $OUT/pytest_edge.log
for i in 1 2; do timeout 600 python bench.py ${BENCH_ARGS:-} > $OUT/bench_e2e_$i.json 2> $OUT/bench_e2e_$i.err; echo "bench rc=$?"; done
python - <<'PY'
import json
for i in (1, 2):
    d = json.loads(open(f"gpurun_out/bench_e2e_{i}.json").readline())
    print(d["value"], d["e2e"], d.get("parity_spot_check"))
PY
python - <<'PY' > $OUT/expand_probe.txt 2>&1
import time, numpy as np, torch
from paper_2503_10855_b200 import _lib
lib = _lib.load()
frames, px = 16, 1080 * 1920
fw = (px + 31) // 32
bits = torch.randint(0, 2**31, (frames, fw), dtype=torch.int32).pin_memory()
out = torch.empty((frames, px), dtype=torch.float32).pin_memory()
for th in (1, 0):
    for r in range(3):
        t = time.perf_counter(); lib.jb_bits_expand_f32(bits.data_ptr(), frames, px, out.data_ptr(), th); dt = time.perf_counter() - t
    print(f"threads={th}: {frames*px*4/dt/1e9:.1f} GB/s of f32 output ({dt*1e3:.2f} ms per 16 frames)")
PY
cat $OUT/expand_probe.txt
