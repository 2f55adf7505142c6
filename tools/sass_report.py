#!/usr/bin/env python
"""Per-opcode instruction / memory mix and the stall hot spots of one kernel
from an `ncu --set full --import-source on` report (SASS source page).

  python tools/sass_report.py report.ncu-rep [units] [--json out.json]

units: work units of the captured launch (e.g. output pixels) for per-unit
counts.  Stalls are the sampled warp states (All Samples) by reason."""
import collections
import csv
import json
import subprocess
import sys


def num(x):
    try:
        return float(x.replace(",", ""))
    except (ValueError, AttributeError):
        return 0.0


def main():
    rep = sys.argv[1]
    units = float(sys.argv[2]) if len(sys.argv) > 2 and not sys.argv[2].startswith("--") else 0.0
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    r = list(csv.reader(out.splitlines()))
    kernel = r[0][1] if r and len(r[0]) > 1 else "?"
    hdr, rows = r[1], r[2:]
    ix = {h: i for i, h in enumerate(hdr)}
    stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    per_op = collections.defaultdict(lambda: collections.Counter())
    stalls = collections.Counter()
    tot_samples = 0
    for x in rows:
        t = x[ix["Source"]].split()
        if not t:
            continue
        op = (t[1] if t[0].startswith("@") else t[0]).split(".")[0]
        c = per_op[op]
        c["warp_inst"] += num(x[ix["Instructions Executed"]])
        for key, col in (("l1_tag_global", "L1 Tag Requests Global"),
                         ("l1_wf_shared", "L1 Wavefronts Shared"),
                         ("l1_wf_shared_ideal", "L1 Wavefronts Shared Ideal"),
                         ("l2_sectors", "L2 Theoretical Sectors Global")):
            if col in ix:  # absent when the kernel has no such access
                c[key] += num(x[ix[col]])
        c["samples"] += num(x[ix["Warp Stall Sampling (All Samples)"]])
        tot_samples += num(x[ix["Warp Stall Sampling (All Samples)"]])
        for s in stall_cols:
            stalls[s[6:]] += num(x[ix[s]])
    res = {"kernel": kernel, "units": units}
    tot = sum(c["warp_inst"] for c in per_op.values())
    res["warp_inst"] = tot
    if units:
        res["thread_inst_per_unit"] = round(tot * 32 / units, 1)
    ops = sorted(per_op.items(), key=lambda kv: -kv[1]["warp_inst"])
    res["ops"] = {k: {q: (round(v / units * 32, 2) if units and q == "warp_inst" else
                          round(v / units, 3) if units else v)
                      for q, v in c.items() if v} for k, c in ops[:28]}
    st = sum(stalls.values()) or 1
    res["stall_share"] = {k: round(v / st, 3) for k, v in stalls.most_common(10) if v}
    hot = sorted(rows, key=lambda x: -num(x[ix["Warp Stall Sampling (All Samples)"]]))[:14]
    res["hot"] = []
    for x in hot:
        why = sorted(((num(x[ix[s]]), s[6:]) for s in stall_cols), reverse=True)[:2]
        res["hot"].append("%5.1f%% %-52s %s" % (
            100 * num(x[ix["Warp Stall Sampling (All Samples)"]]) / max(tot_samples, 1),
            x[ix["Source"]][:52], ",".join("%s:%d" % (n, v) for v, n in why if v)))
    if "--json" in sys.argv:
        with open(sys.argv[sys.argv.index("--json") + 1], "w") as f:
            json.dump(res, f, indent=1)
    print("kernel", kernel, "warp inst", tot, "per unit", res.get("thread_inst_per_unit"))
    for k, c in list(res["ops"].items())[:20]:
        print("  %-10s %s" % (k, c))
    print("stalls", res["stall_share"])
    for h in res["hot"]:
        print(" ", h)


if __name__ == "__main__":
    main()
