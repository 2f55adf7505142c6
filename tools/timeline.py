#!/usr/bin/env python
"""DAG schedule timeline of one C2 execution (device-resident and with host
transfers): python tools/timeline.py [c2]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2006_01201_b200 as fs  # noqa: E402
import fs_synthetic as S  # noqa: E402


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
    lay = {"c1": S.c1_pair, "c2": S.c2_panorama, "c3": S.c3_large_parallax, "c4": S.c4_ring}[cfg](0)
    plan = fs.Plan(lay.dims, lay.offsets, lay.canvas_w, lay.canvas_h, fs.FlowParams(levels=lay.levels))
    plan.execute_host(lay.views, None)
    # the bench's host formats: RGB8 views when all valid, RGB8 canvas when covered
    import numpy as np
    rgb_in = all(bool((v[..., 3] == 255).all()) for v in lay.views)
    cov = np.zeros((lay.canvas_h, lay.canvas_w), bool)
    for v, (x, y) in zip(lay.views, lay.offsets):
        cov[y:y + v.shape[0], x:x + v.shape[1]] |= v[..., 3] >= 128
    rgb_out = rgb_in and bool(cov.all())
    plan.set_host_format(3 if rgb_in else 4, 3 if rgb_out else 4)
    pin = [torch.from_numpy(np.ascontiguousarray(v[..., :3]) if rgb_in else v).pin_memory()
           for v in lay.views]
    out = torch.empty((lay.canvas_h, lay.canvas_w, 3 if rgb_out else 4),
                      dtype=torch.uint8).pin_memory()
    dev = plan.timeline()
    host = plan.timeline([t.data_ptr() for t in pin], out.data_ptr())
    gdev = plan.timeline_graph()
    ghost = plan.timeline_graph([t.data_ptr() for t in pin], out.data_ptr())
    print(json.dumps({"device": dev, "host": host, "graph_device": gdev, "graph_host": ghost},
                     indent=1))


if __name__ == "__main__":
    main()
