#!/usr/bin/env python
"""Per-kernel totals of an ncu launch list (--metrics gpu__time_duration.sum
--csv) of bench.py: python tools/launch_summary.py launches.csv "<command>"."""
import collections
import csv
import json
import sys


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    hdr = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    H = rows[hdr]
    ix = {k: i for i, k in enumerate(H)}
    per = collections.defaultdict(lambda: {"launches": 0, "total_us": 0.0})
    for r in rows[hdr + 1:]:
        if len(r) < len(H) or r[ix["Metric Name"]] != "gpu__time_duration.sum":
            continue
        name = r[ix["Kernel Name"]].replace("void ", "").split("(")[0]
        if not name.startswith(("fs::", "launch::")):
            continue
        v = float(r[ix["Metric Value"]].replace(",", ""))
        unit = r[ix["Metric Unit"]]
        us = {"ns": 1e-3, "nsecond": 1e-3, "ms": 1e3, "msecond": 1e3}.get(unit, 1.0) * v
        per[name]["launches"] += 1
        per[name]["total_us"] += us
    tot = sum(p["total_us"] for p in per.values())
    out = {"source": "ncu --metrics gpu__time_duration.sum --clock-control none over `%s` (all fs:: "
                     "launches of the run; cold-cache serialised, compare shares)" % sys.argv[2],
           "fs_launches": sum(p["launches"] for p in per.values()), "total_us": round(tot, 1),
           "per_kernel": {k: {"launches": v["launches"], "total_us": round(v["total_us"], 1),
                              "share": round(v["total_us"] / tot, 4)}
                          for k, v in sorted(per.items(), key=lambda kv: -kv[1]["total_us"])}}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
