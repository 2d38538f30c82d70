timeout 900 python -m pytest tests -m gpu -q -x -k "backprop or bp_" 2>&1 | tail -2
python - <<'PY'
import numpy as np, torch
from paper_2503_10855_b200 import api, workloads as W
import os
args = W.bp_inputs(1 << 20, 16, 1)
r1 = api.backprop(*args)
os.environ["JB_BP_DIRECT"] = "1"
PY
for v in 0 1; do for r in 1 2; do echo -n "[direct=$v] "; JB_BP_DIRECT=$v python bench.py --workload backprop --steps 10 --warmup 3 --no-cpu --e2e-steps 1 | python -c "import sys,json; d=json.loads(sys.stdin.readline()); print(d['value'], d['roofline']['frac'])"; done; done
