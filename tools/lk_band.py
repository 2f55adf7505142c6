#!/usr/bin/env python
"""One bidirectional flow over a C2 band-sized pair (9000x400, 4 levels) through
the C-ABI, for kernel captures: python tools/lk_band.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2006_01201_b200 as fs  # noqa: E402
import fs_synthetic as S  # noqa: E402

h, w = 400, 9000
a = S.value_noise(h, w + 16, 3).astype(np.float32)
l, r = a[:, :w], a[:, 12:w + 12]
L = fs.ImageBuf(l[:, :, None], np.ones((h, w), np.uint8))
R = fs.ImageBuf(r[:, :, None], np.ones((h, w), np.uint8))
for _ in range(2):
    fs.bidirectional_flow(L, R, fs.FlowParams(levels=4))
