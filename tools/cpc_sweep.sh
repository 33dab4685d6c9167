#!/bin/bash
# decode attention chunks-per-CTA sweep (launch list via ncu)
for c in 1 2 4 8; do
  REATTN_DEC_CPC=$c ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:attend_decode \
     --log-file gpurun_out/cpc_$c.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
  python - $c <<'PY'
import csv, sys
from collections import defaultdict
c = sys.argv[1]
rows = list(csv.reader(open(f"gpurun_out/cpc_{c}.csv")))
hdr = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hdr]; ki = h.index("Kernel Name"); vi = h.index("Metric Value")
agg = defaultdict(list)
for r in rows[hdr + 1:]:
    if len(r) > vi: agg[r[ki][:40]].append(float(r[vi].replace(",", "")))
print("cpc", c, {k: round(sum(v) / len(v) / 1000, 2) for k, v in agg.items()})
PY
done
