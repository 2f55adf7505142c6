#!/usr/bin/env python
"""North_star stage 1 measurement: fisheye -> equirectangular remap with
chromaticity gains for the C2 geometry (4 horizontal views 2750x2800 and the
top/bottom bands 9000x1000 on the 9000x4000 canvas), device-resident (tables
and photos in HBM), CUDA events, L2 flushed between steps.  Prints one JSON
line: python tools/remap_bench.py [steps]"""
import ctypes as C
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2006_01201_b200 as fs  # noqa: E402
from paper_2006_01201_b200 import _native as N  # noqa: E402


def main():
    steps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
    W, H = 9000, 4000
    views = [(0, 600, 2750, 2800), (2083, 600, 2750, 2800), (4166, 600, 2750, 2800),
             (6250, 600, 2750, 2800), (0, 0, 9000, 1000), (0, 3000, 9000, 1000)]
    S = 3000  # fisheye photo size (RGBA8), 180-degree lens
    rng = np.random.RandomState(0)
    jobs = []
    for k, (x0, y0, w, h) in enumerate(views):
        yaw = ((x0 + w / 2) / W) * 2 * np.pi - np.pi
        pitch = 0.0 if k < 4 else (1.2 if k == 4 else -1.2)
        cam = fs.FisheyeCamera(width=S, height=S, cx=(S - 1) / 2, cy=(S - 1) / 2, focal=S / np.pi,
                               radius=S / 2, yaw=yaw, pitch=pitch, roll=0.0)
        t = fs.fisheye_map(cam, W, H, x0, y0, w, h)
        photo = torch.from_numpy(rng.randint(0, 256, (S, S, 4)).astype(np.uint8)).cuda()
        jobs.append((photo, torch.from_numpy(t).cuda(), torch.empty((h, w, 4), dtype=torch.uint8,
                                                                    device="cuda"), w, h))
    gains = (C.c_float * 3)(1.05, 1.0, 0.95)  # host array
    s = torch.cuda.current_stream()
    sp = C.c_void_p(s.cuda_stream)

    def run():
        for photo, t, out, w, h in jobs:
            st = N.lib.fs_remap_rgba8(C.c_void_p(photo.data_ptr()), S, S, 4,
                                      C.c_void_p(t.data_ptr()), w, h, gains,
                                      C.c_void_p(out.data_ptr()), sp)
            assert st == 0, N.last_error()

    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for _ in range(3):
        run()
    torch.cuda.synchronize()
    ms = []
    for _ in range(steps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        run()
        b.record(s)
        torch.cuda.synchronize()
        ms.append(a.elapsed_time(b))
    m = statistics.mean(ms)
    px = sum(w * h for _, _, _, w, h in jobs)
    valid = sum(int((j[1][..., 0] >= 0).sum()) for j in jobs)
    # algorithmic bytes: table 8 + out 4 per pixel, each photo read once
    alg = px * 12 + len(jobs) * S * S * 4
    with open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                           "MEASURED_PEAKS.json")) as f:
        peak = float(json.load(f)["hbm_gbs"])
    gbs = alg / (m * 1e-3) / 1e9
    print(json.dumps({"stage": "fisheye remap + chromaticity gains (C2 geometry, 6 views)",
                      "parity": "unpinned (no reference counterpart)",
                      "ms_per_panorama": round(m, 4), "Mpx_per_s": round(px / m / 1e3, 1),
                      "output_mpx": round(px / 1e6, 2), "valid_fraction": round(valid / px, 3),
                      "algorithmic_GBps": round(gbs, 1), "peak_GBps": peak,
                      "frac": round(gbs / peak, 4), "launches": len(jobs)}))


if __name__ == "__main__":
    main()
