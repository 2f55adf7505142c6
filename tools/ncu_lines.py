#!/usr/bin/env python
"""Top CUDA source lines of an ncu report by sampled warp stalls (cuda,sass
view; needs -lineinfo): python tools/ncu_lines.py report.ncu-rep [n]"""
import csv
import subprocess
import sys


def main():
    rep = sys.argv[1]
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source",
                          "cuda,sass"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    res = []
    hdr = None
    fname = "?"
    for r in rows:
        if r and r[0] == "File Path":
            fname = r[1].split("/")[-1]
        elif r and r[0] == "Line No":
            hdr = r
        elif hdr and len(r) == len(hdr) and r[2] == "-":
            d = dict(zip(hdr[4:], r[4:]))
            tot = float(d.get("Warp Stall Sampling (All Samples)", 0) or 0)
            st = [(float(v or 0), k[6:]) for k, v in d.items()
                  if k.startswith("stall_") and "Not Issued" not in k]
            st.sort(reverse=True)
            res.append((tot, fname, r[0], r[1].strip()[:70],
                        float(d.get("Instructions Executed", 0) or 0), st[:2]))
    all_s = sum(x[0] for x in res) or 1
    for tot, f, ln, src, ie, st in sorted(res, reverse=True)[:n]:
        print("%5.1f%% %s:%-4s %-70s %s" % (100 * tot / all_s, f, ln, src,
                                           " ".join("%s:%d" % (k, v) for v, k in st if v)))


if __name__ == "__main__":
    main()
