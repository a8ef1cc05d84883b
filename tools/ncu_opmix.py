#!/usr/bin/env python3
"""Dynamic SASS opcode mix of one kernel in an ncu report (instructions executed per
opcode, from the source page).  usage: python tools/ncu_opmix.py <rep> <kernel-regex> [top]"""
import collections
import csv
import io
import subprocess
import sys


def main():
    rep, k = sys.argv[1], sys.argv[2]
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
    txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--print-source", "sass", "--csv", "-k",
                          f"regex:{k}"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr = rows[1]
    si, ei = hdr.index("Source"), hdr.index("Instructions Executed")
    c = collections.Counter()
    for r in rows[2:]:
        try:
            n = int(r[ei].replace(",", "") or 0)
        except (ValueError, IndexError):
            continue
        op = r[si].strip().split()
        if not op:
            continue
        m = op[0] if not op[0].startswith("@") else op[1]
        c[m.split(".")[0]] += n
    tot = sum(c.values())
    print(f"{k}: {tot} warp-instructions")
    for m, n in c.most_common(top):
        print(f"{m:12s} {n / tot:6.1%}")


if __name__ == "__main__":
    main()
