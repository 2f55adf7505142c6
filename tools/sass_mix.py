#!/usr/bin/env python
"""Opcode mix and stall hot spots of one kernel from an ncu report:
python tools/sass_mix.py report.ncu-rep [units_for_per_unit_counts]"""
import collections
import csv
import subprocess
import sys


def main():
    rep = sys.argv[1]
    units = float(sys.argv[2]) if len(sys.argv) > 2 else 0
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    r = list(csv.reader(out.splitlines()))
    hdr = r[1]
    rows = r[2:]
    i_src = hdr.index("Source")
    i_s = hdr.index("Warp Stall Sampling (All Samples)")
    i_e = hdr.index("Instructions Executed")
    tot = sum(int(x[i_e] or 0) for x in rows)
    print("warp instructions", tot, ("thread instr per unit %.1f" % (tot * 32 / units)) if units else "")
    c = collections.Counter()
    for x in rows:
        t = x[i_src].split()
        if not t:
            continue
        op = t[1] if t[0].startswith("@") else t[0]
        c[op.split(".")[0]] += int(x[i_e] or 0)
    print([(k, round(v * 32 / units, 1) if units else v) for k, v in c.most_common(24)])
    st = sum(int(x[i_s] or 0) for x in rows) or 1
    for x in sorted(rows, key=lambda x: -int(x[i_s] or 0))[:12]:
        print("%5.1f%%  %s" % (int(x[i_s]) / st * 100, x[i_src][:90]))


if __name__ == "__main__":
    main()
