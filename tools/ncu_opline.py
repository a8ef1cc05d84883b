#!/usr/bin/env python3
"""Source lines executing the most instructions of one opcode in an ncu report (the
source page with CUDA + SASS interleaved).
usage: python tools/ncu_opline.py <rep> <kernel-regex> <OPCODE> [top]"""
import collections
import csv
import io
import subprocess
import sys


def main():
    rep, k, opc = sys.argv[1], sys.argv[2], sys.argv[3]
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 15
    txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--print-source", "cuda,sass", "--csv", "-k",
                          f"regex:{k}"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    c = collections.Counter()
    tot, line, ei, fname = 0, None, None, ""
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            ei = r.index("Instructions Executed")
            continue
        if ei is None or r[0] == "Function Name":
            continue
        if r[0]:
            line = f"{fname}:{r[0]}: {r[1][:80]}"
            continue
        try:
            n = int(r[ei].replace(",", "") or 0)
        except (ValueError, IndexError):
            continue
        ins = r[3].strip().split()
        if not ins:
            continue
        m = ins[0] if not ins[0].startswith("@") else ins[1]
        if m.split(".")[0] == opc:
            c[line] += n
            tot += n
    print(f"{opc}: {tot} warp-instructions")
    for ln, n in c.most_common(top):
        print(f"{n / max(tot, 1):6.1%}  {ln}")


if __name__ == "__main__":
    main()
