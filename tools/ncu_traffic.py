#!/usr/bin/env python
"""DRAM traffic per launch of the roofline kernel, from an ncu metrics CSV of
tools/profile_fold.py (its second, serial execution):

  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
      -k regex:k_lk_sweep --csv --log-file lk.csv python tools/profile_fold.py
  python tools/ncu_traffic.py lk.csv > profiles/ncu_traffic.json

The serial pass launches k_lk_sweep fold by fold: the level tensors, then
levels coarse to fine, iterations 0..I-1 (FIRST = k_lk_sweep<3>, later
ITER = <0>); bench.py's "lk_iter" family is level 0's iterations.
"""
import collections
import csv
import json
import sys


def main():
    path = sys.argv[1]
    levels = int(sys.argv[2]) if len(sys.argv) > 2 else 4
    iters = int(sys.argv[3]) if len(sys.argv) > 3 else 3
    rows = list(csv.reader(open(path)))
    hdr = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    H = rows[hdr]
    ix = {k: i for i, k in enumerate(H)}
    launches = collections.OrderedDict()
    for r in rows[hdr + 1:]:
        if len(r) < len(H):
            continue
        key = r[ix["ID"]]
        d = launches.setdefault(key, {"name": r[ix["Kernel Name"]]})
        d[r[ix["Metric Name"]]] = float(r[ix["Metric Value"]].replace(",", ""))
    seq = list(launches.values())
    # split schedule: per fold, the level tensors (levels x k_lk_sweep<2>),
    # then per level (coarse to fine) FIRST (<3>) and iters-1 ITER (<0>)
    per_fold = levels + levels * iters
    nfold = len(seq) // 2 // per_fold
    serial = seq[len(seq) - nfold * per_fold:]
    pick = []
    for f in range(nfold):
        base = f * per_fold + levels + (levels - 1) * iters  # level 0's first iteration
        pick += serial[base:base + iters]
    assert all("<" in p["name"] for p in pick)
    rd = sum(p["dram__bytes_read.sum"] for p in pick) / len(pick)
    wr = sum(p["dram__bytes_write.sum"] for p in pick) / len(pick)
    us = sum(p["gpu__time_duration.sum"] for p in pick) / len(pick) / 1e3
    print(json.dumps({
        "kernel": sorted(set(p["name"] for p in pick)),
        "launches": len(pick),
        "lk_iter_dram_bytes_per_launch": round(rd + wr),
        "dram_read_bytes_per_launch": round(rd),
        "dram_write_bytes_per_launch": round(wr),
        "ncu_avg_launch_us (serialised, cold)": round(us, 2),
        "source": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum over the "
                  "level-0 FIRST + ITER launches (bench.py's lk_iter family) of the second, "
                  "serial execution of tools/profile_fold.py c2",
    }, indent=1))


if __name__ == "__main__":
    main()
