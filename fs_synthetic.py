"""Synthetic, seeded stitching workloads (BASELINE.json configs).

Input generation only: numpy, no torch, no GPU and no import of the product
package, so the reference arm of bench.py and the CPU oracle legs build their
inputs without touching the B200 library.  Every arm reads the same bytes.

Texture is multi-octave value noise (octave o = 1..7: cell 2^o px, amplitude
2^(o/2), smoothstep-bilinear lattice drawn from MT19937(seed) in U(-1,1)),
normalised to [0.1, 0.9] and quantised to 8 bits; RGB channels use seeds s,
s+101, s+202.  Views are windows of one scene with a per-view content shift,
which creates the parallax the flow must absorb.  Every view is RGBA8 with
alpha 255 (all valid), the reference's load_image convention
(src/image.cpp:27-43): value = byte * (1.0f/255.0f), valid = alpha >= 128.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List, Tuple

import numpy as np

INV255 = np.float32(1.0) / np.float32(255.0)  # 1.0f/255.0f as the reference computes it


def value_noise(h: int, w: int, seed: int, octaves=range(1, 8)) -> np.ndarray:
    """Multi-octave smoothstep value noise in [0.1, 0.9], float32 (h, w)."""
    rng = np.random.RandomState(seed)
    acc = np.zeros((h, w), np.float32)
    for o in octaves:
        cell = 2 ** o
        amp = np.float32(2.0 ** (o / 2.0))
        ny, nx = h // cell + 1, w // cell + 1  # lattice cells covering the image
        lat = rng.uniform(-1.0, 1.0, size=(ny + 1, nx + 1)).astype(np.float32)
        f = np.arange(cell, dtype=np.float32) / np.float32(cell)
        s = f * f * (3 - 2 * f)  # smoothstep weights, identical for every cell
        # x: each lattice column pair feeds `cell` consecutive pixels
        t = (lat[:, :-1, None] * (1 - s) + lat[:, 1:, None] * s).reshape(ny + 1, nx * cell)
        t = t[:, :w]
        # y: same per lattice row pair, in row blocks (bounded temporaries)
        for r0 in range(0, ny, 64):
            r1 = min(ny, r0 + 64)
            v = (t[r0:r1, None, :] * (1 - s)[None, :, None]
                 + t[r0 + 1:r1 + 1, None, :] * s[None, :, None]).reshape((r1 - r0) * cell, w)
            y0 = r0 * cell
            y1 = min(h, r1 * cell)
            if y1 > y0:
                acc[y0:y1] += amp * v[:y1 - y0]
    lo, hi = float(acc.min()), float(acc.max())
    return (0.1 + 0.8 * (acc - lo) / max(hi - lo, 1e-6)).astype(np.float32)


def rgb_scene(h: int, w: int, seed: int) -> np.ndarray:
    """(h, w, 3) uint8 scene."""
    if h * w >= (1 << 20):  # numpy releases the GIL: one thread per channel
        from concurrent.futures import ThreadPoolExecutor
        with ThreadPoolExecutor(3) as ex:
            chans = list(ex.map(lambda d: value_noise(h, w, seed + d), (0, 101, 202)))
    else:
        chans = [value_noise(h, w, seed + d) for d in (0, 101, 202)]
    return np.clip(np.rint(np.stack(chans, axis=-1) * 255.0), 0, 255).astype(np.uint8)


def rgba(view_rgb: np.ndarray) -> np.ndarray:
    out = np.empty(view_rgb.shape[:2] + (4,), np.uint8)
    out[..., :3] = view_rgb
    out[..., 3] = 255
    return out


@dataclass
class Layout:
    """Ordered placements on a fixed canvas (pipeline.hpp:15-27), 8-bit views."""
    name: str
    canvas_w: int
    canvas_h: int
    views: List[np.ndarray]             # (h, w, 4) uint8 RGBA, fold order
    offsets: List[Tuple[int, int]]
    levels: int = 4
    truth: dict = field(default_factory=dict)

    @property
    def dims(self) -> List[Tuple[int, int]]:
        return [(v.shape[1], v.shape[0]) for v in self.views]

    @property
    def canvas_mpx(self) -> float:
        return self.canvas_w * self.canvas_h / 1e6

    def float_views(self):
        """(data float32 (h,w,3), valid uint8 (h,w)) per view, as load_image makes them."""
        out = []
        for v in self.views:
            data = v[..., :3].astype(np.float32) * INV255
            out.append((np.ascontiguousarray(data), (v[..., 3] >= 128).astype(np.uint8)))
        return out


def c1_pair(seed: int = 0, size: int = 1024, parallax: int = 12) -> Layout:
    """configs[0]: two size x size views, R placed at size/2 showing content
    shifted by `parallax` px: FlowLtoR = (-parallax, 0), FlowRtoL = (+parallax, 0)."""
    half = size // 2
    scene = rgb_scene(size, size + half + parallax, seed)
    left = scene[:, 0:size]
    right = scene[:, half + parallax: half + parallax + size]
    return Layout("C1 pair %dx%d, %d px parallax" % (size, size, parallax), size + half, size,
                  [rgba(left), rgba(right)], [(0, 0), (half, 0)], 4,
                  {"ltor": (-parallax, 0.0), "rtol": (parallax, 0.0)})


def c2_panorama(seed: int = 0, parallax: int = 12) -> Layout:
    """configs[1]: 4 horizontal views (2750x2800 at x = 0, 2083, 4166, 6250,
    y = 600, content shifted by `parallax`*k) + top/bottom bands (9000x1000 at
    y = 0 and y = 3000) folded onto a 9000x4000 canvas, views first."""
    W, H = 9000, 4000
    xs = [0, 2083, 4166, 6250]
    scene = rgb_scene(H, W + parallax * len(xs), seed)
    views, offs = [], []
    for k, x in enumerate(xs):
        c0 = x + parallax * k
        views.append(rgba(scene[600:3400, c0:c0 + 2750]))
        offs.append((x, 600))
    views.append(rgba(scene[0:1000, 0:W]))
    offs.append((0, 0))
    views.append(rgba(scene[3000:4000, 0:W]))
    offs.append((0, 3000))
    return Layout("C2 9000x4000 panorama: 4 views + top/bottom bands", W, H, views, offs, 4)


def c3_large_parallax(seed: int = 0, bg: int = 8, fg: int = 80) -> Layout:
    """configs[2]: 2048x1024 views, R at x = 1024; background disparity `bg`,
    a 600x500 foreground block at `fg` px disparity; levels = 6."""
    H, Wv = 1024, 2048
    back = rgb_scene(H, 3072 + bg + fg, seed)
    front = rgb_scene(H, 3072 + bg + fg, seed + 7)
    left = back[:, 0:Wv].copy()
    right = back[:, 1024 + bg:1024 + bg + Wv].copy()
    fy, fx, fh, fw = 262, 1224, 500, 600       # block in canvas coords (inside the overlap)
    left[fy:fy + fh, fx:fx + fw] = front[fy:fy + fh, fx:fx + fw]
    rx = fx - 1024 - fg                        # R shows the block shifted by fg
    right[fy:fy + fh, rx:rx + fw] = front[fy:fy + fh, fx:fx + fw]
    return Layout("C3 large parallax (%d px bg, %d px block)" % (bg, fg), 3072, H,
                  [rgba(left), rgba(right)], [(0, 0), (1024, 0)], 6)


def c4_ring(seed: int = 0, parallax: int = 12) -> Layout:
    """configs[3]: 8 views 2560x6144 at x = 2048k, y = 1024 on 16384x8192
    (7 planar seams of 512x6144; the wrap-around seam is out of scope)."""
    W, H = 16384, 8192
    scene = rgb_scene(6144, W + 2560 + parallax * 8, seed)
    views, offs = [], []
    for k in range(8):
        x = min(2048 * k, W - 2560)
        c0 = x + parallax * k
        views.append(rgba(scene[:, c0:c0 + 2560]))
        offs.append((x, 1024))
    return Layout("C4 16384x8192 8-view ring", W, H, views, offs, 4)


def small_strip(seed: int = 0, n: int = 3, vw: int = 180, vh: int = 150, step: int = 120,
                parallax: int = 3) -> Layout:
    """Small multi-view strip (test-sized C2 analogue)."""
    W = step * (n - 1) + vw
    scene = rgb_scene(vh, W + parallax * n, seed)
    views, offs = [], []
    for k in range(n):
        x = step * k
        c0 = x + parallax * k
        views.append(rgba(scene[:, c0:c0 + vw]))
        offs.append((x, 0))
    return Layout("strip", W, vh, views, offs, 3)


def small_panorama(seed: int = 0, parallax: int = 4) -> Layout:
    """C2 geometry scaled by 1/10 (900x400): 4 views + 2 bands."""
    W, H = 900, 400
    xs = [0, 208, 416, 625]
    scene = rgb_scene(H, W + parallax * len(xs), seed)
    views, offs = [], []
    for k, x in enumerate(xs):
        c0 = x + parallax * k
        views.append(rgba(scene[60:340, c0:c0 + 275]))
        offs.append((x, 60))
    views.append(rgba(scene[0:100, 0:W]))
    offs.append((0, 0))
    views.append(rgba(scene[300:400, 0:W]))
    offs.append((0, 300))
    return Layout("C2/10 900x400 panorama", W, H, views, offs, 3)


def tile_panorama(seed: int = 0, parallax: int = 6) -> Layout:
    """C2's geometry at 2048x800 (levels 4): 4 views 620x560 at y = 120 and
    two 2048x200 bands whose 2048x80 Area3 boxes cross every seam — the layout
    the row/column flow tiles (fs_plan_set_tiling) are tested on."""
    W, H = 2048, 800
    xs = [0, 476, 952, 1428]
    scene = rgb_scene(H, W + parallax * len(xs), seed)
    views, offs = [], []
    for k, x in enumerate(xs):
        c0 = x + parallax * k
        views.append(rgba(scene[120:680, c0:c0 + 620]))
        offs.append((x, 120))
    views.append(rgba(scene[0:200, 0:W]))
    offs.append((0, 0))
    views.append(rgba(scene[600:800, 0:W]))
    offs.append((0, 600))
    return Layout("C2 geometry 2048x800 (tile tests)", W, H, views, offs, 4)
