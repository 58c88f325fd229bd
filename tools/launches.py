#!/usr/bin/env python
"""Summarise an ncu --csv launch list (gpu__time_duration.sum, optionally
dram__bytes_read.sum / dram__bytes_write.sum) per kernel name.
usage: launches.py <file.csv> [reps]"""
import collections
import csv
import sys

lines = open(sys.argv[1]).read().splitlines()
start = [i for i, l in enumerate(lines) if l.startswith('"ID"')][0]
rows = list(csv.reader(lines[start:]))
hdr = rows[0]
ii, ki, mi, vi, ui = (hdr.index(k) for k in ("ID", "Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
mult = {"nsecond": 1.0, "ns": 1.0, "usecond": 1e3, "us": 1e3, "msecond": 1e6, "ms": 1e6,
        "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
launch = collections.OrderedDict()
for r in rows[1:]:
    k = r[ki].split("(")[0].split("::")[-1][:44]
    launch.setdefault((int(r[ii]), k), {})[r[mi]] = float(r[vi].replace(",", "")) * mult.get(r[ui], 1.0)
agg = collections.OrderedDict()
for (_, k), m in launch.items():
    a = agg.setdefault(k, [0, 0.0, 0.0, 0.0])
    a[0] += 1
    a[1] += m.get("gpu__time_duration.sum", 0.0)
    a[2] += m.get("dram__bytes_read.sum", 0.0)
    a[3] += m.get("dram__bytes_write.sum", 0.0)
tot = sum(a[1] for a in agg.values())
print(f"{'kernel':44s} {'n':>4s} {'us/launch':>10s} {'share':>6s} {'MB rd':>9s} {'MB wr':>9s} {'GB/s':>7s}")
for k, (n, t, rd, wr) in agg.items():
    print(f"{k:44s} {n:4d} {t / n / 1e3:10.1f} {t / tot * 100:5.1f}% {rd / n / 1e6:9.1f} {wr / n / 1e6:9.1f} "
          f"{(rd + wr) / t if t else 0:7.1f}")
print(f"total {tot / 1e6 / reps:.3f} ms per rep ({reps} reps)")
