#!/usr/bin/env python
"""Dump dense_pyr_lk / bidirectional_flow outputs of a fixed case list to an
.npz, to compare two builds bit for bit (kernel rewrites that must not change
a single float, e.g. the smoothing kernels).

usage: python tools/flow_bits.py out.npz          # dump
       python tools/flow_bits.py a.npz b.npz      # compare
"""
import sys

import os

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

CASES = [((64, 64), dict(levels=3, window_radius=5, iterations_per_level=3)),
         ((128, 128), dict()), ((96, 160), dict(smoothing_passes=0)),
         ((80, 72), dict(smoothing_passes=1, iterations_per_level=1)),
         ((200, 90), dict(smoothing_passes=3, window_radius=3)),
         ((256, 512), dict(levels=5)), ((9, 700), dict(levels=1)),
         ((700, 9), dict(levels=1)), ((131, 257), dict(smoothing_passes=4)),
         ((1000, 1500), dict()), ((400, 9000), dict())]


def dump(path):
    import paper_2006_01201_b200.api as fs
    import fs_synthetic as S
    out = {}
    for k, ((h, w), kw) in enumerate(CASES):
        base = S.value_noise(h + 40, w + 40, seed=w + k)
        frm = base[20:20 + h, 20:20 + w]
        to = base[17:17 + h, 25:25 + w]
        one = np.ones((h, w), np.uint8)
        f = fs.dense_pyr_lk(fs.ImageBuf(frm, one), fs.ImageBuf(to, one),
                            fs.FlowParams(**kw))
        out[f"vec{k}"], out[f"valid{k}"] = f.vec, f.valid
    np.savez(path, **out)


def compare(a, b):
    A, B = np.load(a), np.load(b)
    bad = [k for k in A.files if not np.array_equal(A[k].view(np.uint8), B[k].view(np.uint8))]
    print("bit-identical" if not bad else f"DIFFER: {bad}")
    return not bad


if __name__ == "__main__":
    if len(sys.argv) == 2:
        dump(sys.argv[1])
    else:
        sys.exit(0 if compare(sys.argv[1], sys.argv[2]) else 1)
