#!/bin/bash
# One GPU round: parity tests, a bench line, and the per-kernel launch list (ncu).
# usage (under gpurun): bash tools/gpu_check.sh TAG [pytest -k expr]
TAG=${1:-run}; K=${2:-"not 1m"}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -k "$K" > gpurun_out/pytest_$TAG.log 2>&1
echo "pytest_rc=$? $(tail -1 gpurun_out/pytest_$TAG.log)"
timeout 600 python bench.py --steps 300 --warmup 10 --no-cpu-baseline > gpurun_out/bench_$TAG.log 2>&1
echo "bench_rc=$?"
python - "$TAG" <<'PY'
import json, sys
t = sys.argv[1]
d = json.loads(open(f"gpurun_out/bench_{t}.log").read().strip().splitlines()[-1])
print("step_us", round(d["value"], 1), "scan_us", round(d["roofline"]["launch_us"], 1),
      "scan_frac", round(d["roofline"]["frac"], 3), "e2e_us", round(d["e2e"]["value"], 1),
      "kernels", d["kernels_per_step"], "clk", d["clocks"])
PY
python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/plain_$TAG.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline \
    > gpurun_out/ncu_$TAG.log 2>&1
echo "ncu_rc=$?"
python - "$TAG" <<'PY'
import csv, sys
from collections import defaultdict
t = sys.argv[1]
rows = list(csv.reader(open(f"gpurun_out/launches_{t}.csv")))
hdr = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hdr]; ki = h.index("Kernel Name"); vi = h.index("Metric Value")
agg = defaultdict(list)
for r in rows[hdr + 1:]:
    if len(r) > vi:
        agg[r[ki][:80]].append(float(r[vi].replace(",", "")))
for k, v in agg.items():
    print(f"{len(v):4d} {sum(v) / len(v) / 1000:10.2f} us  {k}")
PY
