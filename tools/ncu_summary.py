#!/usr/bin/env python
"""Summarise an .ncu-rep (ncu --set full) into the numbers DESIGN.md and
profiles/ cite: duration, DRAM traffic, occupancy, issue rate, top stalls.

usage: python tools/ncu_summary.py report.ncu-rep [--json out.json]
"""
import csv
import io
import json
import subprocess
import sys
from collections import OrderedDict

WANT = OrderedDict([
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_pct"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_pct"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy_pct"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "fp64_pipe_pct"),
    ("smsp__inst_executed.sum", "warp_insts"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue_active_pct"),
])


def raw(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for vals in rows[2:]:
        d = OrderedDict()
        d["kernel"] = vals[hdr.index("Kernel Name")][:60]
        for m, k in WANT.items():
            if m in hdr:
                i = hdr.index(m)
                d[k] = (vals[i], units[i])
        stalls = []
        # warps stalled per issue-active cycle, by reason (this ncu's names;
        # older versions: smsp__average_warp_latency_issue_stalled_*)
        for pre, post in (("smsp__average_warps_issue_stalled_", "_per_issue_active.ratio"),
                          ("smsp__average_warp_latency_issue_stalled_", ".ratio")):
            for i, h in enumerate(hdr):
                if h.startswith(pre) and h.endswith(post):
                    try:
                        stalls.append((float(vals[i].replace(",", "")), h[len(pre):-len(post)]))
                    except ValueError:
                        pass
            if stalls:
                break
        stalls.sort(reverse=True)
        d["top_stalls_cycles_per_issue"] = [(n, round(v, 2)) for v, n in stalls[:6]]
        res.append(d)
    return res


def to_bytes(v):
    val, unit = v
    f = float(val.replace(",", ""))
    return f * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)


if __name__ == "__main__":
    res = raw(sys.argv[1])
    for d in res:
        print(json.dumps(d))
    if "--json" in sys.argv:
        out = sys.argv[sys.argv.index("--json") + 1]
        with open(out, "w") as f:
            json.dump(res, f, indent=1)
