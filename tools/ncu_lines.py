#!/usr/bin/env python3
"""Per-source-line instruction / stall breakdown of one kernel in an ncu report.
usage: python tools/ncu_lines.py <report.ncu-rep> <kernel-substring> [top]"""
import collections
import csv
import io
import os
import re
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    rep, kname = sys.argv[1], sys.argv[2]
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
    txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--print-source", "sass", "--csv", "-k",
                          f"regex:{kname}"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr = rows[1]
    ai, ei, wi = hdr.index("Address"), hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
    ins = []
    for r in rows[2:]:
        try:
            ins.append((int(r[ai], 16), int(r[ei].replace(",", "") or 0), int(r[wi].replace(",", "") or 0)))
        except (ValueError, IndexError):
            pass
    base = min(a for a, _, _ in ins)
    with tempfile.TemporaryDirectory() as d:
        subprocess.run(["cuobjdump", "-xelf", "all", os.path.join(ROOT, "paper_2409_17346_b200", "libdmtz.so")],
                       cwd=d, capture_output=True)
        cub = [f for f in os.listdir(d) if f.endswith(".cubin")][0]
        sass = subprocess.run(["nvdisasm", "-g", os.path.join(d, cub)], capture_output=True, text=True).stdout
    # the function whose text section holds as many instructions as the report
    best = None
    for m in re.finditer(r"\n\s*\.text\.([^:\s]+):", sass):
        if kname.split("<")[0].replace("regex:", "") not in m.group(1):
            continue
        j = sass.find("\n\t.section", m.end())
        body = sass[m.end(): j if j > 0 else len(sass)]
        n = len(re.findall(r"\n\s+/\*[0-9a-f]{4,}\*/", body))
        if best is None or abs(n - len(ins)) < abs(best[0] - len(ins)):
            best = (n, body)
    off2line, line = {}, None
    for ln in best[1].splitlines():
        m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
        if m:
            line = (m.group(1), int(m.group(2)))
            continue
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/", ln)
        if m and line:
            off2line[int(m.group(1), 16)] = line
    tot = sum(n for _, n, _ in ins)
    stt = sum(w for _, _, w in ins) or 1
    byl, stl = collections.Counter(), collections.Counter()
    for a, n, w in ins:
        ln = off2line.get(a - base, ("?", 0))
        byl[ln] += n
        stl[ln] += w
    print(f"{kname}: {tot} warp-instructions, {len(ins)} SASS lines")
    for ln, n in sorted(byl.items(), key=lambda x: -(x[1] / tot + stl[x[0]] / stt))[:top]:
        code = ""
        if os.path.exists(ln[0]):
            code = open(ln[0]).read().splitlines()[ln[1] - 1].strip()[:72]
        print(f"{n / tot:6.1%} stall {stl[ln] / stt:6.1%}  {os.path.basename(str(ln[0]))[:16]}:{ln[1]:<4d} {code}")


if __name__ == "__main__":
    main()
