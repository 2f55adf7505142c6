#!/usr/bin/env python
"""One serial (non-graph) execution of the C2 fold with per-kernel CUDA-event
timing — a deterministic launch order for targeted ncu captures:

  per fold k = 1..5: partition, check_box, crop_gray, pyramid x3,
                     then for levels 3..0: lk_prep, k_lk_sweep x3, smooth;
                     edt x3, blend, compose
  e.g. band fold 4, level 0, later iterations: -k regex:k_lk_sweep -s 46 -c 2
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2006_01201_b200 as fs  # noqa: E402
import fs_synthetic as S  # noqa: E402


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
    lay = {"c1": S.c1_pair, "c2": S.c2_panorama, "c3": S.c3_large_parallax, "c4": S.c4_ring}[cfg](0)
    plan = fs.Plan(lay.dims, lay.offsets, lay.canvas_w, lay.canvas_h, fs.FlowParams(levels=lay.levels))
    plan.execute_host(lay.views, None)
    stats, total = plan.profile()
    print(json.dumps({"total_ms": total, "kernels": stats}))


if __name__ == "__main__":
    main()
