#!/usr/bin/env python3
"""Summarise ncu --set full reports into profiles/ncu_summary.json + a text table.
usage: python tools/ncu_summary.py <workload-label> <report.ncu-rep> [...]"""
import csv
import io
import json
import os
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "launch__registers_per_thread", "lts__t_sector_hit_rate.pct"]
SCALE = {"us": 1e-6, "ms": 1e-3, "ns": 1e-9, "B": 1, "KB": 1e3, "MB": 1e6, "GB": 1e9, "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3,
         "second": 1}


def main():
    label, reps = sys.argv[1], sys.argv[2:]
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = os.path.join(root, "profiles", "ncu_summary.json")
    data = json.load(open(out)) if os.path.exists(out) else {}
    entry = data.setdefault(label, {})
    for rep in reps:
        txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        rows = list(csv.reader(io.StringIO(txt)))
        hdr, units = rows[0], rows[1]
        for r in rows[2:]:
            name = r[hdr.index("Kernel Name")].split("(")[0].split("<")[0].replace("void ", "").replace("dmtz::", "")
            d = {}
            for k in KEYS:
                if k in hdr:
                    i = hdr.index(k)
                    try:
                        v = float(r[i].replace(",", "")) * SCALE.get(units[i], 1)
                    except ValueError:
                        continue
                    d[k] = v
            d["dram_bytes"] = d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)
            d["report"] = os.path.basename(rep)
            entry.setdefault(name, d) if name not in entry else entry.__setitem__(name + "@" + os.path.basename(rep), d)
            print(f"{label:18s} {name:14s} t={d.get('gpu__time_duration.sum', 0) * 1e3:9.3f} ms "
                  f"dram={d['dram_bytes'] / 1e9:7.3f} GB alu={d.get('sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active', 0):5.1f}% "
                  f"issue={d.get('smsp__issue_active.avg.pct_of_peak_sustained_active', 0):5.1f}% "
                  f"warps={d.get('sm__warps_active.avg.pct_of_peak_sustained_active', 0):5.1f}% "
                  f"regs={d.get('launch__registers_per_thread', 0):.0f}  [{os.path.basename(rep)}]")
    json.dump(data, open(out, "w"), indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
