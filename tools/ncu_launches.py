#!/usr/bin/env python
"""Quick per-kernel table of an ncu --csv launch list (gpu__time_duration.sum, optionally dram__bytes_read.sum):
per kernel name, launches, total / mean time and, when present, achieved read bandwidth."""
import collections
import csv
import sys


def main(path, top=25):
    hdr, launches = None, collections.OrderedDict()
    for r in csv.reader(open(path)):
        if r and r[0] == "ID":
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        key = (d["ID"], d["Kernel Name"])
        launches.setdefault(key, {})[d["Metric Name"]] = (float(d["Metric Value"].replace(",", "")),
                                                         d["Metric Unit"])
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for (_, name), m in launches.items():
        t, unit = m["gpu__time_duration.sum"]
        t = t * {"ns": 1e-9, "usecond": 1e-6, "us": 1e-6, "msecond": 1e-3, "ms": 1e-3}.get(unit, 1e-9)
        b = 0.0
        if "dram__bytes_read.sum" in m:
            v, u = m["dram__bytes_read.sum"]
            b = v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
        a = agg[name[:90]]
        a[0] += 1
        a[1] += t
        a[2] += b
    tot = sum(a[1] for a in agg.values())
    print(f"{'n':>5} {'total ms':>9} {'mean us':>8} {'share':>6} {'GB/s':>7}  kernel")
    for k, (n, t, b) in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
        print(f"{n:5d} {t*1e3:9.3f} {t/n*1e6:8.2f} {t/tot:6.1%} {b/t/1e9 if b else 0:7.0f}  {k}")


if __name__ == "__main__":
    main(sys.argv[1])
