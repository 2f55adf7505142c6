#!/usr/bin/env python
"""Segment 0 of one rank of the sharded C4 schedule, run 3 times (for an ncu
launch list): python tools/shard_rank_profile.py N RANK [c4|c2]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2006_01201_b200 as fs  # noqa: E402
import fs_synthetic as S  # noqa: E402
from paper_2006_01201_b200.shard import ShardedPlan  # noqa: E402

n, r = int(sys.argv[1]), int(sys.argv[2])
cfg = sys.argv[3] if len(sys.argv) > 3 else "c4"
lay = {"c2": S.c2_panorama, "c4": S.c4_ring}[cfg](0)
plan = fs.Plan(lay.dims, lay.offsets, lay.canvas_w, lay.canvas_h, fs.FlowParams(levels=lay.levels),
               views_rgba=lay.views)
sp = ShardedPlan(plan, n, r)
for _ in range(3):
    sp.execute_segment(0)
torch.cuda.synchronize()
