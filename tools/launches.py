#!/usr/bin/env python
"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list."""
import collections
import csv
import sys

lines = open(sys.argv[1]).read().splitlines()
start = [i for i, l in enumerate(lines) if l.startswith('"ID"')][0]
rows = list(csv.reader(lines[start:]))
hdr = rows[0]
ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
agg = collections.OrderedDict()
scale = {"nsecond": 1.0, "ns": 1.0, "usecond": 1e3, "us": 1e3, "msecond": 1e6, "ms": 1e6}
for r in rows[1:]:
    k = r[ki].split("(")[0].split("::")[-1][:48]
    agg.setdefault(k, []).append(float(r[vi].replace(",", "")) * scale[r[ui]])
tot = sum(sum(v) for v in agg.values())
print(f"{'kernel':48s} {'launches':>8s} {'mean us':>10s} {'share':>6s}")
for k, v in agg.items():
    print(f"{k:48s} {len(v):8d} {sum(v) / len(v) / 1e3:10.1f} {sum(v) / tot * 100:5.1f}%")
print(f"total {tot / 1e6 / reps:.3f} ms per rep ({reps} reps)")
