"""TEST INFRASTRUCTURE — numpy restatement of the fisheye pre-processing
(north_star stage 1: distortion remap + chromaticity gains).

PARITY UNPINNED: the reference has no such stage (SPEC.md:12 leaves
pre-processing to Hugin/PanoTools), so there is no
reference code, golden vector or known-answer test to pin this restatement
to.  It restates the camera model documented in include/fs_b200.h
(equidistant fisheye r = f * theta, camera = Ry(yaw) Rx(pitch) Rz(roll),
equirectangular canvas spanning 360 x 180 degrees) and the remap's float32
arithmetic, operation for operation.  Only tests/ may import it.
"""
import numpy as np


def rotation(yaw, pitch, roll):
    cy, sy = np.cos(yaw), np.sin(yaw)
    cp, sp = np.cos(pitch), np.sin(pitch)
    cr, sr = np.cos(roll), np.sin(roll)
    Ry = np.array([[cy, 0, sy], [0, 1, 0], [-sy, 0, cy]])
    Rx = np.array([[1, 0, 0], [0, cp, -sp], [0, sp, cp]])
    Rz = np.array([[cr, -sr, 0], [sr, cr, 0], [0, 0, 1]])
    return Ry @ Rx @ Rz


def fisheye_map(cam, canvas_w, canvas_h, x0, y0, w, h):
    """(h, w, 2) float32 source positions, (-1, -1) where invalid (float64 math)."""
    R = rotation(cam["yaw"], cam["pitch"], cam["roll"])
    v, u = np.mgrid[0:h, 0:w].astype(np.float64)
    lat = np.pi / 2 - ((y0 + v) + 0.5) / canvas_h * np.pi
    lon = ((x0 + u) + 0.5) / canvas_w * (2 * np.pi) - np.pi
    d = np.stack([np.cos(lat) * np.sin(lon), np.sin(lat), np.cos(lat) * np.cos(lon)], -1)
    dc = d @ R  # R^T d for row vectors
    dx, dy, dz = dc[..., 0], dc[..., 1], dc[..., 2]
    theta = np.arccos(np.clip(dz, -1.0, 1.0))
    r = cam["focal"] * theta
    rho = np.sqrt(dx * dx + dy * dy)
    safe = np.where(rho > 0, rho, 1.0)
    sx = np.where(rho > 0, cam["cx"] + r * (dx / safe), cam["cx"])
    sy = np.where(rho > 0, cam["cy"] - r * (dy / safe), cam["cy"])
    ok = (r <= cam["radius"]) & (sx >= 0) & (sy >= 0) & (sx <= cam["width"] - 1) & \
        (sy <= cam["height"] - 1)
    out = np.full((h, w, 2), -1.0, np.float32)
    out[..., 0] = np.where(ok, sx, -1.0).astype(np.float32)
    out[..., 1] = np.where(ok, sy, -1.0).astype(np.float32)
    return out


def remap_rgba8(src, table, gains=(1.0, 1.0, 1.0)):
    """The kernel's float32 bilinear gather + gains, in its operation order."""
    f32 = np.float32
    sh, sw, ch = src.shape
    mx, my = table[..., 0].astype(f32), table[..., 1].astype(f32)
    ok = (mx >= 0) & (my >= 0) & (mx <= f32(sw - 1)) & (my <= f32(sh - 1))
    x0 = np.floor(np.where(ok, mx, 0)).astype(np.int64)
    y0 = np.floor(np.where(ok, my, 0)).astype(np.int64)
    x1 = np.minimum(x0 + 1, sw - 1)
    y1 = np.minimum(y0 + 1, sh - 1)
    fx = (np.where(ok, mx, 0) - x0.astype(f32)).astype(f32)
    fy = (np.where(ok, my, 0) - y0.astype(f32)).astype(f32)
    one = f32(1.0)
    w00 = (one - fx) * (one - fy)
    w10 = fx * (one - fy)
    w01 = (one - fx) * fy
    w11 = fx * fy
    out = np.zeros(table.shape[:2] + (4,), np.uint8)
    for c in range(3):
        p = src[..., c].astype(f32)
        v = ((w00 * p[y0, x0] + w10 * p[y0, x1]) + w01 * p[y1, x0]) + w11 * p[y1, x1]
        r = np.floor(v * f32(gains[c]) + f32(0.5)).astype(f32)
        out[..., c] = np.where(ok, np.minimum(r, f32(255.0)), 0).astype(np.uint8)
    out[..., 3] = np.where(ok, 255, 0).astype(np.uint8)
    return out


def render_fisheye(scene, cam):
    """Synthetic fisheye photo of an equirectangular scene (H x W x 3 uint8):
    each fisheye pixel looks up the scene direction it sees (nearest) — used
    for round-trip checks."""
    R = rotation(cam["yaw"], cam["pitch"], cam["roll"])
    H, W = scene.shape[:2]
    yy, xx = np.mgrid[0:cam["height"], 0:cam["width"]].astype(np.float64)
    px, py = xx - cam["cx"], cam["cy"] - yy
    r = np.sqrt(px * px + py * py)
    theta = r / cam["focal"]
    safe = np.where(r > 0, r, 1.0)
    dc = np.stack([np.sin(theta) * px / safe, np.sin(theta) * py / safe, np.cos(theta)], -1)
    d = dc @ R.T
    lat = np.arcsin(np.clip(d[..., 1], -1, 1))
    lon = np.arctan2(d[..., 0], d[..., 2])
    u = np.clip(((lon + np.pi) / (2 * np.pi) * W - 0.5).round().astype(int), 0, W - 1)
    v = np.clip(((np.pi / 2 - lat) / np.pi * H - 0.5).round().astype(int), 0, H - 1)
    img = scene[v, u]
    img[r > cam["radius"]] = 0
    return img


def chroma_gains(views, offsets, canvas_w, canvas_h):
    """(n, 3) gains: exact integer overlap sums against each pixel's first
    covering earlier view, chained from view 0 (float64 on the host)."""
    n = len(views)
    owner = np.full((canvas_h, canvas_w), 255, np.int64)
    for k, (v, (x, y)) in enumerate(zip(views, offsets)):
        h, w = v.shape[:2]
        sub = owner[y:y + h, x:x + w]
        sub[(sub == 255) & (v[..., 3] >= 128)] = k
    g = np.ones((n, 3), np.float64)
    for k in range(1, n):
        v, (x, y) = views[k], offsets[k]
        h, w = v.shape[:2]
        own = owner[y:y + h, x:x + w]
        valid = v[..., 3] >= 128
        num = np.zeros(3)
        den = np.zeros(3)
        for m in range(k):
            sel = valid & (own == m)
            if not sel.any():
                continue
            vm, (xm, ym) = views[m], offsets[m]
            yy, xx = np.nonzero(sel)
            q = vm[yy + y - ym, xx + x - xm, :3].astype(np.int64).sum(0)
            p = v[yy, xx, :3].astype(np.int64).sum(0)
            num += g[m] * q.astype(np.float64)
            den += p.astype(np.float64)
        g[k] = np.where(den > 0, num / np.where(den > 0, den, 1), 1.0)
    return g.astype(np.float32)
