#!/usr/bin/env python3
"""Per-kernel totals of an ncu --metrics gpu__time_duration.sum --csv launch list.
usage: python tools/launch_table.py <launches.csv> [top]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 20
hdr, agg = None, collections.defaultdict(lambda: [0, 0.0])
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if not hdr or len(r) < len(hdr):
        continue
    d = dict(zip(hdr, r))
    if d.get("Metric Name") != "gpu__time_duration.sum":
        continue
    name = d["Kernel Name"].split("(")[0].replace("void ", "").replace("dmtz::", "")
    v = float(d["Metric Value"].replace(",", ""))
    unit = d.get("Metric Unit", "")
    ms = v / 1e6 if unit in ("nsecond", "ns") else v / 1e3 if unit in ("usecond", "us") else v
    agg[name][0] += 1
    agg[name][1] += ms
tot = sum(v[1] for v in agg.values())
for k, v in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
    print(f"{k:36s} {v[0]:5d} {v[1]:10.3f} ms {v[1] / tot:6.1%}")
print(f"{'total':36s} {sum(v[0] for v in agg.values()):5d} {tot:10.3f} ms")
