#!/usr/bin/env python
"""One device-resident execution of a config's plan (for kernel captures):
python tools/plan_once.py [c2|c1|c3|c4] [n_exec]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2006_01201_b200 as fs  # noqa: E402
import fs_synthetic as S  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 1
lay = {"c1": S.c1_pair, "c2": S.c2_panorama, "c3": S.c3_large_parallax, "c4": S.c4_ring}[cfg](0)
plan = fs.Plan(lay.dims, lay.offsets, lay.canvas_w, lay.canvas_h, fs.FlowParams(levels=lay.levels))
for _ in range(n):
    plan.execute_host(lay.views, None)
plan.close()
