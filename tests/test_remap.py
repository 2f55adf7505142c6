"""Fisheye distortion remap + chromaticity gains (north_star stage 1;
SURVEY.md §8(f) rank 2).  PARITY UNPINNED: the reference has no such stage,
so the library is checked against the numpy restatement in oracle/remap.py
(the table within float rounding of an independent float64 evaluation, the
GPU remap bit-exact on the same table) and by a render -> remap round trip."""
import numpy as np
import pytest

import fs_synthetic as S


def _cam(fs, **kw):
    c = dict(width=640, height=640, cx=319.5, cy=319.5, focal=640 / np.pi, radius=320.0,
             yaw=0.3, pitch=-0.1, roll=0.05)
    c.update(kw)
    return fs.FisheyeCamera(**c), c


def test_fisheye_map_matches_restatement():
    import paper_2006_01201_b200 as fs
    from oracle import remap as R
    for kw in ({}, dict(yaw=-2.0, pitch=0.4, roll=-0.3), dict(cx=300.25, cy=333.0, radius=250.0)):
        cam, c = _cam(fs, **kw)
        W, H = 2000, 1000
        # the camera looks at lon = yaw: the rectangle around it
        x0 = int((c["yaw"] + np.pi) / (2 * np.pi) * W) - 160
        t = fs.fisheye_map(cam, W, H, x0, 340, 320, 320)
        o = R.fisheye_map(c, W, H, x0, 340, 320, 320)
        valid_t, valid_o = t[..., 0] >= 0, o[..., 0] >= 0
        assert valid_t.mean() > 0.3
        # validity may differ only where the ray grazes the image circle
        assert (valid_t != valid_o).mean() < 1e-3
        both = valid_t & valid_o
        assert np.abs(t[both] - o[both]).max() < 2e-4


def test_fisheye_map_contracts():
    import paper_2006_01201_b200 as fs
    cam, _ = _cam(fs, focal=-1.0)
    with pytest.raises(fs.ContractError):
        fs.fisheye_map(cam, 100, 50, 0, 0, 10, 10)


@pytest.mark.gpu
@pytest.mark.parametrize("channels", [3, 4])
def test_remap_bit_exact_random_tables(fs, channels):
    from oracle import remap as R
    rng = np.random.RandomState(channels)
    src = rng.randint(0, 256, (97, 131, channels)).astype(np.uint8)
    h, w = 60, 77
    t = np.stack([rng.uniform(-3, 133, (h, w)), rng.uniform(-3, 99, (h, w))], -1).astype(np.float32)
    t[::7, ::5] = np.floor(t[::7, ::5])          # integer positions
    t[3, :10] = [130.0, 96.0]                    # the last column / row exactly
    t[4, :10] = -1.0                             # invalid marker
    for gains in ((1.0, 1.0, 1.0), (1.3, 0.8, 2.5), (0.0, 1.0, 0.5)):
        got = fs.remap_rgba8(src, t, gains)
        want = R.remap_rgba8(src, t, gains)
        assert np.array_equal(got, want)


@pytest.mark.gpu
def test_remap_round_trip(fs):
    """Render a fisheye photo of an equirectangular scene, remap it back onto
    the canvas: the interior reproduces the scene (up to resampling)."""
    from oracle import remap as R
    W, H = 1200, 600
    scene = S.rgb_scene(H, W, 4)  # uint8 RGB
    cam, c = _cam(fs, width=800, height=800, cx=399.5, cy=399.5, focal=800 / np.pi, radius=400.0,
                  yaw=0.5, pitch=0.0, roll=0.0)
    photo = R.render_fisheye(scene, c)
    x0 = int((c["yaw"] + np.pi) / (2 * np.pi) * W) - 100
    t = fs.fisheye_map(cam, W, H, x0, 200, 200, 200)
    view = fs.remap_rgba8(photo, t, (1.0, 1.0, 1.0))
    assert np.array_equal(view, R.remap_rgba8(photo, t))
    ok = view[..., 3] == 255
    assert ok.mean() > 0.99
    diff = np.abs(view[..., :3].astype(int) - scene[200:400, x0:x0 + 200].astype(int))[ok]
    assert diff.mean() < 12.0
    # gains scale the colours (chromaticity correction)
    g = fs.remap_rgba8(photo, t, (0.5, 1.0, 1.0))
    assert np.array_equal(g, R.remap_rgba8(photo, t, (0.5, 1.0, 1.0)))
    assert g[..., 0][ok].mean() < 0.6 * view[..., 0][ok].mean() + 1


@pytest.mark.gpu
def test_chroma_gains_match_restatement(fs):
    """Views of one scene with per-view exposure factors: the estimated gains
    equal the restatement's (exact integer sums) and undo the exposure."""
    from oracle import remap as R
    lay = S.small_panorama(seed=3)
    expo = [(1.0, 1.0, 1.0), (0.8, 0.9, 1.1), (1.2, 1.0, 0.85), (0.9, 1.1, 1.0),
            (1.05, 0.95, 1.0), (0.95, 1.0, 1.05)][:len(lay.views)]
    views = []
    for v, e in zip(lay.views, expo):
        w = v.copy()
        w[..., :3] = np.clip(np.rint(v[..., :3] * np.array(e)), 0, 255).astype(np.uint8)
        views.append(w)
    got = fs.chroma_gains(views, lay.offsets, lay.canvas_w, lay.canvas_h)
    want = R.chroma_gains(views, lay.offsets, lay.canvas_w, lay.canvas_h)
    assert np.array_equal(got, want)
    assert np.allclose(got[1], 1.0 / np.array(expo[1]), rtol=0.03)
    assert np.array_equal(got[0], [1, 1, 1])
