#!/usr/bin/env python
"""C4 end-to-end diagnostics: the plan's transfer bytes, its e2e time, and the
raw PCIe time of the same bytes (one pinned H2D / D2H copy each, alone and
together): python tools/c4_d2h_diag.py [cfg]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2006_01201_b200 as fs  # noqa: E402
import fs_synthetic as S  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
lay = {"c2": S.c2_panorama, "c4": S.c4_ring}[cfg](0)
plan = fs.Plan(lay.dims, lay.offsets, lay.canvas_w, lay.canvas_h, fs.FlowParams(levels=lay.levels))
plan.execute_host(lay.views, None)
rgb_in = all(bool((v[..., 3] == 255).all()) for v in lay.views)
cov = np.zeros((lay.canvas_h, lay.canvas_w), bool)
for v, (x, y) in zip(lay.views, lay.offsets):
    cov[y:y + v.shape[0], x:x + v.shape[1]] |= v[..., 3] >= 128
rgb_out = rgb_in and bool(cov.all())
plan.set_host_format(3 if rgb_in else 4, 3 if rgb_out else 4)
h2d, d2h = plan.transfer_bytes()
hv = [torch.from_numpy(np.ascontiguousarray(v[..., :3]) if rgb_in else v).pin_memory() for v in lay.views]
ho = torch.empty((lay.canvas_h, lay.canvas_w, 3 if rgb_out else 4), dtype=torch.uint8).pin_memory()
ptrs = [t.data_ptr() for t in hv]
for _ in range(3):
    plan.execute_ptrs(ptrs, ho.data_ptr())
ts = []
for _ in range(5):
    t0 = time.perf_counter()
    plan.execute_ptrs(ptrs, ho.data_ptr())
    ts.append((time.perf_counter() - t0) * 1e3)
print(cfg, "rgb_in", rgb_in, "rgb_out", rgb_out, "h2d MB", h2d / 1e6, "d2h MB", d2h / 1e6,
      "e2e ms", [round(t, 2) for t in ts])
dev = torch.empty(max(h2d, d2h), dtype=torch.uint8, device="cuda")
hin = torch.empty(h2d, dtype=torch.uint8).pin_memory()
hout = torch.empty(d2h, dtype=torch.uint8).pin_memory()
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for name, up, down in (("h2d", True, False), ("d2h", False, True), ("both", True, True)):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    if up:
        with torch.cuda.stream(s1):
            dev[:h2d].copy_(hin, non_blocking=True)
    if down:
        with torch.cuda.stream(s2):
            hout.copy_(dev[:d2h], non_blocking=True)
    torch.cuda.synchronize()
    print("raw", name, round((time.perf_counter() - t0) * 1e3, 2), "ms")
plan.close()
