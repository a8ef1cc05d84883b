#!/usr/bin/env python3
"""Per-kernel launch list + DRAM traffic of one step from a single ncu pass:
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
      --clock-control none --csv --log-file step.csv python tools/profile_once.py C4
usage: python tools/ncu_step.py <workload-label> step.csv [out.txt]
Writes '<kernel>@step' entries (launches, mean time and DRAM bytes per launch) into
profiles/ncu_summary.json and prints the launch table."""
import collections
import csv
import json
import os
import sys

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3,
         "second": 1, "B": 1, "KB": 1e3, "MB": 1e6, "GB": 1e9, "ns": 1e-9, "us": 1e-6, "ms": 1e-3}


def main():
    label, path = sys.argv[1], sys.argv[2]
    rows = list(csv.reader(open(path)))
    hdr, launches = None, collections.OrderedDict()
    for r in rows:
        if "Kernel Name" in r and "Metric Name" in r:
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        name = d["Kernel Name"].split("(")[0].split("<")[0].replace("void ", "").replace("dmtz::", "")
        v = float(d["Metric Value"].replace(",", "")) * SCALE.get(d["Metric Unit"], 1)
        launches.setdefault(d["ID"], {"name": name})[d["Metric Name"]] = v
    per = collections.defaultdict(lambda: {"n": 0, "t": 0.0, "dram": 0.0})
    for L in launches.values():
        p = per[L["name"]]
        p["n"] += 1
        p["t"] += L.get("gpu__time_duration.sum", 0.0)
        p["dram"] += L.get("dram__bytes_read.sum", 0.0) + L.get("dram__bytes_write.sum", 0.0)
    tot = sum(p["t"] for p in per.values()) or 1.0
    lines = [f"{'kernel':24s} {'n':>5s} {'total ms':>10s} {'share':>7s} {'avg us':>10s} {'dram MB/launch':>15s}"]
    for k, p in sorted(per.items(), key=lambda x: -x[1]["t"]):
        lines.append(f"{k:24s} {p['n']:5d} {p['t'] * 1e3:10.2f} {p['t'] / tot:7.1%} {p['t'] / p['n'] * 1e6:10.1f} "
                     f"{p['dram'] / p['n'] / 1e6:15.2f}")
    txt = "\n".join(lines)
    print(txt)
    if len(sys.argv) > 3:
        open(sys.argv[3], "w").write(f"# {label}: ncu launch list of one step (cold caches, serialised)\n{txt}\n")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = os.path.join(root, "profiles", "ncu_summary.json")
    data = json.load(open(out)) if os.path.exists(out) else {}
    entry = data.setdefault(label, {})
    for k, p in per.items():
        entry[k + "@step"] = {"launches": p["n"], "time_s_per_launch": p["t"] / p["n"],
                              "dram_bytes": p["dram"] / p["n"], "share_of_kernel_time": p["t"] / tot,
                              "source": os.path.basename(path)}
    json.dump(data, open(out, "w"), indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
