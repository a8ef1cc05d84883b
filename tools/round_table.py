#!/usr/bin/env python3
"""Per-round kernel times from an ncu launch list of one dmtz_correct call (profile mode).
usage: python tools/round_table.py launches.csv"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h, out = None, []
for r in rows:
    if "Kernel Name" in r:
        h = r
        continue
    if h and len(r) == len(h):
        d = dict(zip(h, r))
        out.append((d["Kernel Name"].split("(")[0].split("<")[0].replace("void ", ""), float(d["Metric Value"]) / 1e3))
tot = collections.Counter()
for n, t in out:
    tot[n] += t
print({k: round(v / 1e3, 2) for k, v in tot.most_common()}, "ms")
per = collections.defaultdict(list)
for n, t in out:
    per[n].append(t)
names = ["k_screen", "k_decode", "k_edit_rows", "k_units_from_bits", "k_loop_check"]
print("round " + " ".join(f"{n[2:]:>12s}" for n in names))
for i in range(len(per["k_screen"])):
    if i < 20 or i % 10 == 0:
        print(f"{i + 1:5d} " + " ".join(f"{per[n][i]:12.1f}" if i < len(per[n]) else " " * 12 for n in names))
print("16+   " + " ".join(f"{sum(per[n][15:]):12.1f}" for n in names))
