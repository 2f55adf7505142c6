"""CPU: the synthetic workloads have the geometry BASELINE.json / SURVEY.md
§8(d) specify and are deterministic."""
import numpy as np

import fs_synthetic as S


def test_value_noise_range_and_determinism():
    a = S.value_noise(64, 80, 3)
    b = S.value_noise(64, 80, 3)
    assert a.dtype == np.float32 and np.array_equal(a, b)
    assert abs(a.min() - 0.1) < 1e-6 and abs(a.max() - 0.9) < 1e-6
    assert not np.array_equal(a, S.value_noise(64, 80, 4))


def test_small_layouts():
    lay = S.small_panorama(1)
    assert (lay.canvas_w, lay.canvas_h) == (900, 400) and len(lay.views) == 6
    for v, (x, y) in zip(lay.views, lay.offsets):
        assert v.dtype == np.uint8 and v.shape[2] == 4 and np.all(v[..., 3] == 255)
        assert x + v.shape[1] <= lay.canvas_w and y + v.shape[0] <= lay.canvas_h
    d, valid = lay.float_views()[0]
    assert d.dtype == np.float32 and valid.all()
    # value = byte * (1.0f/255.0f), src/image.cpp:31-37
    assert d[0, 0, 0] == np.float32(lay.views[0][0, 0, 0]) * (np.float32(1) / np.float32(255))


def test_c1_geometry_and_truth():
    lay = S.c1_pair(0, size=128, parallax=12)
    assert (lay.canvas_w, lay.canvas_h) == (192, 128)
    assert lay.offsets == [(0, 0), (64, 0)]
    l, r = lay.views[0][..., :3], lay.views[1][..., :3]
    # R's content at canvas x equals L's content at x + 12 over the overlap
    assert np.array_equal(r[:, 0:128 - 64 - 12], l[:, 64 + 12:128])
