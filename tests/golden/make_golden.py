#!/usr/bin/env python
"""Generate tests/golden/golden_v1.npz: small input/output vectors produced by
the REFERENCE itself (oracle/_ref/libfsref.so, compiled from
/root/reference/proj/src by oracle/Makefile with the reference's Release
flags).  The fixtures let the oracle restatement and the GPU path be pinned
on machines where the reference cannot be built (e.g. the GPU box).

    python tests/golden/make_golden.py        # rewrites golden_v1.npz
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import reference  # noqa: E402
import fs_synthetic as S  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden_v1.npz")


def main():
    ref = reference()
    ref.set_threads(1)
    g = {}
    # 1. fold of a 3-view strip (pipeline.cpp:150-204 without metrics)
    lay = S.small_strip(seed=11, n=3, vw=64, vh=40, step=44, parallax=2)
    fv = lay.float_views()
    params = (3, 5, 2, 1e-4, 2)
    out, ov = ref.stitch_placed([d for d, _ in fv], [v for _, v in fv], lay.offsets, lay.canvas_w,
                                lay.canvas_h, params)
    for k, (d, v) in enumerate(fv):
        g["strip_view%d" % k] = d
        g["strip_valid%d" % k] = v
    g["strip_offsets"] = np.array(lay.offsets, np.int32)
    g["strip_canvas"] = np.array([lay.canvas_w, lay.canvas_h], np.int32)
    g["strip_params"] = np.array(params, np.float64)
    g["strip_out"] = out
    g["strip_out_valid"] = ov
    # 2. dense_pyr_lk, default params, shifted texture
    base = S.value_noise(60, 76, 5)
    frm, to = base[6:54, 8:72].copy(), base[4:52, 5:69].copy()
    vec, val = ref.dense_pyr_lk(frm, to, (4, 8, 3, 1e-4, 2))
    g["lk_from"], g["lk_to"], g["lk_vec"], g["lk_valid"] = frm, to, vec, val
    # 3. exact EDT of a random mask
    rng = np.random.RandomState(2024)
    m = (rng.randint(0, 7, size=(23, 31)) == 0).astype(np.uint8)
    m[5, 7] = 1
    g["edt_mask"], g["edt_out"] = m, ref.distance_transform(m)
    # 4. Eq. 1 on two overlapping rectangles
    ml = np.zeros((20, 34), np.uint8)
    mr = np.zeros((20, 34), np.uint8)
    ml[1:19, :22] = 1
    mr[3:20, 12:] = 1
    label, counts = ref.compute_partition(ml, mr)
    g["bf_label"], g["bf_counts"], g["bf_out"] = label, counts, ref.compute_blend(label, counts)
    # 5. Code 1 on random flows
    h, w = 24, 32
    L = np.stack([S.value_noise(h, w, 30 + c) for c in range(3)], -1)
    R = np.stack([S.value_noise(h, w, 40 + c) for c in range(3)], -1)
    vl = np.ones((h, w), np.uint8)
    vr = np.ones((h, w), np.uint8)
    vl[:, 21:] = 0
    vr[:, :10] = 0
    lab, cnt = ref.compute_partition(vl, vr)
    b = ref.compute_blend(lab, cnt)
    flr = rng.uniform(-5, 5, size=(h, w, 2)).astype(np.float32)
    frl = rng.uniform(-5, 5, size=(h, w, 2)).astype(np.float32)
    F, FV = ref.blend_pair(L, vl, R, vr, flr, frl, b, lab)
    g.update(bp_L=L, bp_vl=vl, bp_R=R, bp_vr=vr, bp_flr=flr, bp_frl=frl, bp_b=b, bp_label=lab,
             bp_out=F, bp_out_valid=FV)
    # 6. pyramid
    img = S.value_noise(37, 29, 9)
    pyr = ref.build_pyramid(img, 4)
    g["pyr_in"] = img
    for k, lv in enumerate(pyr):
        g["pyr_l%d" % k] = lv
    np.savez_compressed(OUT, **g)
    print("wrote", OUT, os.path.getsize(OUT), "bytes")


if __name__ == "__main__":
    main()
