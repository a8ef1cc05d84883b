#!/usr/bin/env python3
"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list."""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 5]
hdr, rows = rows[0], rows[1:]
ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
seq = [(r[ki].split("(")[0].split("<")[0].replace("void ", "").replace("dmtz::", "")[-28:],
        float(r[vi].replace(",", "")) * scale[r[ui]]) for r in rows]
tot, cnt = collections.defaultdict(float), collections.Counter()
for k, v in seq:
    tot[k] += v
    cnt[k] += 1
T = sum(tot.values())
print(f"{'kernel':30s} {'n':>5s} {'total ms':>10s} {'share':>6s} {'avg us':>10s}")
for k in sorted(tot, key=lambda k: -tot[k]):
    print(f"{k:30s} {cnt[k]:5d} {tot[k] / 1e3:10.2f} {tot[k] / T:6.1%} {tot[k] / cnt[k]:10.1f}")
if "-v" in sys.argv:
    for k, v in seq:
        print(f"  {k:28s} {v:10.1f}")
