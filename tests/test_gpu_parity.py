"""GPU parity: every C-ABI entry point against the CPU oracle restatement
(oracle/fs_oracle.c, itself pinned bit-exact to the compiled reference in
test_oracle.py) on identical seeded inputs.

Tolerances (BASELINE.json north_star):
  * integer / index / mask work (labels, counts, boxes, pyramid dims, squared
    distances, valid bits): bit-exact;
  * pyramid, gray, crop, EDT, Eq. 1: bit-exact (same fp32/fp64 op order, no FMA);
  * flow: identical valid bits, mean EPE <= 1e-4 px (spec: <= 0.05 px);
  * blend (fp32 output of fp64 math; exp() may differ by 1 ulp): |d| <= 1e-6;
  * 8-bit output: +-1 LSB on >= 99.9% of pixels (in practice 100%).
"""
import numpy as np
import pytest

import fs_synthetic as S

pytestmark = pytest.mark.gpu

EPE_TOL = 1e-4


def _img(fs, data, valid=None):
    data = np.asarray(data, np.float32)
    if data.ndim == 2:
        data = data[:, :, None]
    if valid is None:
        valid = np.ones(data.shape[:2], np.uint8)
    return fs.ImageBuf(data, valid)


def _rgb(h, w, seed):
    return np.stack([S.value_noise(h, w, seed + d) for d in (0, 101, 202)], -1)


def _epe(a, b):
    return float(np.sqrt(((a - b) ** 2).sum(-1)).mean())


# ---------------------------------------------------------------- imagecore
def test_to_gray_bit_exact(fs, oracle):
    d = _rgb(37, 53, 1)
    g = fs.to_gray(_img(fs, d))
    assert np.array_equal(g.data[..., 0], oracle.to_gray(d))
    one = S.value_noise(9, 11, 2)
    assert np.array_equal(fs.to_gray(_img(fs, one)).data[..., 0], one)


def test_bilinear_sample_matches(fs, oracle):
    rng = np.random.RandomState(3)
    d = _rgb(20, 30, 4)
    v = (rng.rand(20, 30) > 0.3).astype(np.uint8)
    img = _img(fs, d, v)
    xy = rng.uniform(-5, 35, size=(400, 2))
    got = fs.bilinear_sample_batch(img, xy)
    exp = np.stack([oracle.bilinear_sample(d, v, x, y) for x, y in xy])
    assert np.array_equal(got, exp)
    # reference KATs (test_image.cpp:268-301)
    two = _img(fs, np.array([[0.2, 0.6]], np.float32))
    assert fs.bilinear_sample(two, 0.5, 0.0)[0] == pytest.approx(0.4)
    one_invalid = _img(fs, np.array([[0.3, 0.9]], np.float32), np.array([[1, 0]], np.uint8))
    assert fs.bilinear_sample(one_invalid, 0.75, 0.0)[0] == pytest.approx(0.3)
    none_valid = _img(fs, np.array([[0.3, 0.9]], np.float32), np.array([[0, 0]], np.uint8))
    assert fs.bilinear_sample(none_valid, 0.5, 0.0)[0] == 0.0


@pytest.mark.parametrize("shape", [(1, 10), (13, 9), (64, 80), (3, 1)])
def test_partition_and_crop_bit_exact(fs, oracle, shape):
    rng = np.random.RandomState(sum(shape))
    h, w = shape
    ml = (rng.rand(h, w) > 0.4).astype(np.uint8)
    mr = (rng.rand(h, w) > 0.4).astype(np.uint8)
    part = fs.compute_partition(fs.Mask(ml), fs.Mask(mr))
    lab, cnt = oracle.compute_partition(ml, mr)
    assert np.array_equal(part.label, lab)
    assert np.array_equal(part.counts, cnt)
    d = _rgb(h, w, 5)
    if cnt[3] == 0:
        with pytest.raises(fs.EmptyRegionError):
            fs.crop_overlap(_img(fs, d, ml), part)
        return
    c = fs.crop_overlap(_img(fs, d, ml), part)
    od, ov, off = oracle.crop_overlap(d, ml, lab, cnt)
    assert (c.offset_x, c.offset_y) == off
    assert np.array_equal(c.image.data, od)
    assert np.array_equal(c.image.valid, ov)


def test_partition_kats(fs):
    # test_image.cpp:331-366
    def cols(w, h, c0, c1):
        m = np.zeros((h, w), np.uint8)
        m[:, c0:c1 + 1] = 1
        return fs.Mask(m)
    p = fs.compute_partition(cols(10, 2, 0, 3), cols(10, 2, 6, 9))
    assert list(p.counts) == [4, 8, 8, 0]
    p = fs.compute_partition(cols(10, 1, 0, 6), cols(10, 1, 4, 9))
    assert list(p.label[0]) == [1, 1, 1, 1, 3, 3, 3, 2, 2, 2]
    with pytest.raises(fs.ContractError):
        fs.compute_partition(fs.Mask(np.zeros((3, 3), np.uint8)), fs.Mask(np.zeros((3, 4), np.uint8)))


def test_place_on_canvas(fs, oracle):
    d = _rgb(7, 5, 9)
    v = np.ones((7, 5), np.uint8)
    v[2, 3] = 0
    c = fs.place_on_canvas(_img(fs, d, v), 6, 2, 20, 12)
    od, ov = oracle.place_on_canvas(d, v, 6, 2, 20, 12)
    assert np.array_equal(c.data, od) and np.array_equal(c.valid, ov)
    with pytest.raises(fs.LayoutError):
        fs.place_on_canvas(_img(fs, d, v), 16, 0, 20, 12)
    with pytest.raises(fs.LayoutError):
        fs.place_on_canvas(_img(fs, d, v), -1, 0, 20, 12)


# ---------------------------------------------------------------- pyramid + flow
@pytest.mark.parametrize("shape,levels", [((16, 16), 2), ((20, 20), 5), ((37, 53), 4),
                                          ((129, 67), 6), ((8, 300), 4)])
def test_build_pyramid_bit_exact(fs, oracle, shape, levels):
    g = S.value_noise(*shape, seed=shape[0])
    got = fs.build_pyramid(_img(fs, g), levels)
    exp = oracle.build_pyramid(g, levels)
    assert len(got) == len(exp)
    for a, b in zip(got, exp):
        assert np.array_equal(a.data[..., 0], b)


def test_pyramid_depth_kat(fs):
    # test_flow.cpp:79-84: 20 -> 10, 10/2 = 5 < 8
    assert len(fs.build_pyramid(_img(fs, S.value_noise(20, 20, 3)), 5)) == 2
    with pytest.raises(fs.ContractError):
        fs.build_pyramid(_img(fs, _rgb(16, 16, 4)), 2)


LK_CASES = [
    ((64, 64), (3.0, 0.0), dict(levels=3, window_radius=5, iterations_per_level=3)),
    ((128, 128), (5.0, 3.0), dict()),
    ((96, 160), (-4.0, 1.5), dict(smoothing_passes=0)),
    ((80, 72), (2.0, -1.0), dict(smoothing_passes=1, iterations_per_level=1)),
    ((200, 90), (1.0, 2.0), dict(smoothing_passes=3, window_radius=3)),
    ((256, 512), (-12.0, 0.0), dict(levels=5)),
]


@pytest.mark.parametrize("shape,shift,kw", LK_CASES)
def test_dense_pyr_lk_matches_oracle(fs, oracle, shape, shift, kw):
    h, w = shape
    base = S.value_noise(h + 40, w + 40, seed=w)
    frm = base[20:20 + h, 20:20 + w]
    sx, sy = int(round(shift[0])), int(round(shift[1]))
    to = base[20 - sy:20 - sy + h, 20 - sx:20 - sx + w]
    p = fs.FlowParams(**kw)
    f = fs.dense_pyr_lk(_img(fs, frm), _img(fs, to), p)
    vec, valid = oracle.dense_pyr_lk(frm, to, p)
    assert np.array_equal(f.valid, valid)
    assert _epe(f.vec, vec) <= EPE_TOL
    assert np.abs(f.vec - vec).max() <= 1e-2


def test_lk_reference_kats(fs):
    # zero-motion fixpoint (test_flow.cpp:91-102)
    img = _img(fs, S.value_noise(48, 48, 21))
    f = fs.dense_pyr_lk(img, img, fs.FlowParams(levels=3, window_radius=5))
    assert np.sqrt((f.vec ** 2).sum(-1)).max() <= 1e-3
    # textureless -> zero and invalid (test_flow.cpp:126-137)
    flat = _img(fs, np.full((32, 32), 0.7, np.float32))
    f = fs.dense_pyr_lk(flat, flat, fs.FlowParams(levels=2))
    assert np.all(f.vec == 0.0) and np.all(f.valid == 0)
    # contract checks (test_flow.cpp:139-146)
    with pytest.raises(fs.ContractError):
        fs.dense_pyr_lk(img, _img(fs, S.value_noise(48, 24, 1)))
    with pytest.raises(fs.ContractError):
        fs.dense_pyr_lk(img, img, fs.FlowParams(levels=0))


def test_bidirectional_flow_matches_oracle(fs, oracle):
    L = _rgb(120, 90, 11)
    R = np.roll(L, (1, 4), axis=(0, 1))
    lr, rl = fs.bidirectional_flow(_img(fs, L), _img(fs, R))
    (olr, olv), (orl, orv) = oracle.bidirectional_flow(L, R)
    assert np.array_equal(lr.valid, olv) and np.array_equal(rl.valid, orv)
    assert _epe(lr.vec, olr) <= EPE_TOL and _epe(rl.vec, orl) <= EPE_TOL
    m = lr.vec[20:-20, 20:-20].mean((0, 1))
    assert m[0] == pytest.approx(4.0, abs=0.3) and m[1] == pytest.approx(1.0, abs=0.3)


def test_flow_helpers(fs, oracle):
    rng = np.random.RandomState(17)
    vec = rng.uniform(-10, 10, size=(4, 5, 2)).astype(np.float32)
    ff = fs.FlowField(vec, np.ones((4, 5), np.uint8))
    assert np.array_equal(fs.flow_magnitude(ff), oracle.flow_magnitude(vec))
    e = fs.embed_flow(ff, 5, 7, 20, 15)
    ov, oval = oracle.embed_flow(vec, np.ones((4, 5), np.uint8), 5, 7, 20, 15)
    assert np.array_equal(e.vec, ov) and np.array_equal(e.valid, oval)
    with pytest.raises(fs.ContractError):
        fs.embed_flow(ff, 19, 0, 20, 15)


# ---------------------------------------------------------------- EDT + Eq. 1
@pytest.mark.parametrize("shape,density,seed", [((8, 8), 0.0, 0), ((37, 51), 1 / 7, 1),
                                                ((1, 60), 0.1, 2), ((60, 1), 0.1, 3),
                                                ((200, 31), 0.002, 4), ((31, 300), 0.01, 5),
                                                ((128, 128), 0.3, 6)])
def test_distance_transform_bit_exact(fs, oracle, shape, density, seed):
    rng = np.random.RandomState(seed)
    m = (rng.rand(*shape) < density).astype(np.uint8)
    m[rng.randint(shape[0]), rng.randint(shape[1])] = 1
    d = fs.distance_transform(fs.Mask(m))
    assert np.array_equal(d.d, oracle.distance_transform(m))


def test_distance_transform_kats(fs):
    m = np.zeros((8, 8), np.uint8)
    m[0, 0] = 1
    d = fs.distance_transform(fs.Mask(m)).d
    assert d[4, 3] == 5.0 and d[0, 0] == 0.0 and d[0, 7] == 7.0
    with pytest.raises(fs.EmptyRegionError):
        fs.distance_transform(fs.Mask(np.zeros((4, 4), np.uint8)))


def _rect_masks(w, h, rng):
    lx1 = w // 2 + rng.randint(w // 2)
    rx0 = rng.randint(lx1 - 1)
    l = np.zeros((h, w), np.uint8)
    r = np.zeros((h, w), np.uint8)
    l[rng.randint(4):h - rng.randint(4), :lx1 + 1] = 1
    r[rng.randint(4):h - rng.randint(4), rx0:] = 1
    return l, r


def test_compute_blend_bit_exact(fs, oracle):
    rng = np.random.RandomState(7)
    for _ in range(10):
        l, r = _rect_masks(24 + rng.randint(41), 16 + rng.randint(33), rng)
        part = fs.compute_partition(fs.Mask(l), fs.Mask(r))
        b = fs.compute_blend(part)
        assert np.array_equal(b.b, oracle.compute_blend(part.label, part.counts))
    # 10x1 strip KAT (test_blend_field.cpp:89-96)
    l = np.zeros((1, 10), np.uint8)
    r = np.zeros((1, 10), np.uint8)
    l[0, :7] = 1
    r[0, 4:] = 1
    b = fs.compute_blend(fs.compute_partition(fs.Mask(l), fs.Mask(r))).b[0]
    assert b[4] == pytest.approx(0.25) and b[5] == pytest.approx(0.5) and b[6] == pytest.approx(0.75)
    # empty side -> 0.5 (test_blend_field.cpp:147-159)
    l = np.zeros((4, 8), np.uint8)
    l[:, :6] = 1
    r = l.copy()
    r[:, 6] = 1
    b = fs.compute_blend(fs.compute_partition(fs.Mask(l), fs.Mask(r))).b
    assert np.all(b[:, :6] == 0.5)


# ---------------------------------------------------------------- blender
def test_softmax_kats(fs, oracle):
    sl, sr = fs.softmax_weights(0.75, 0.25, 0.0, 0.0, fs.BlendParams(10.0, 0.37))
    assert sl == pytest.approx(0.99330714907571527, rel=1e-15)
    rng = np.random.RandomState(4)
    for _ in range(200):
        b = rng.rand()
        args = (1 - b, b, rng.rand() * 20, rng.rand() * 20)
        assert fs.softmax_weights(*args) == oracle.softmax_weights(*args)
    sl, sr = fs.softmax_weights(1.0, 0.0, 100.0, 0.0, fs.BlendParams(5000.0))
    assert np.isfinite(sl) and sl == pytest.approx(1.0)


def _overlap_case(fs, oracle, w, h, seed, random_flow=True, mag=6.0):
    L = _rgb(h, w, seed)
    R = _rgb(h, w, seed + 5)
    third = w // 3
    vl = np.ones((h, w), np.uint8)
    vr = np.ones((h, w), np.uint8)
    vl[:, 2 * third:] = 0
    vr[:, :third] = 0
    part = fs.compute_partition(fs.Mask(vl), fs.Mask(vr))
    b = fs.compute_blend(part)
    rng = np.random.RandomState(seed + 11)
    if random_flow:
        flr = rng.uniform(-mag, mag, size=(h, w, 2)).astype(np.float32)
        frl = rng.uniform(-mag, mag, size=(h, w, 2)).astype(np.float32)
    else:
        flr = np.zeros((h, w, 2), np.float32)
        frl = np.zeros((h, w, 2), np.float32)
    return L, vl, R, vr, part, b, flr, frl


def test_blend_pair_matches_oracle(fs, oracle):
    for seed in (10, 20, 30):
        L, vl, R, vr, part, b, flr, frl = _overlap_case(fs, oracle, 128, 128, seed)
        ones = np.ones(part.label.shape, np.uint8)
        F = fs.blend_pair(_img(fs, L, vl), _img(fs, R, vr), fs.FlowField(flr, ones),
                          fs.FlowField(frl, ones), b, part)
        OF, OV = oracle.blend_pair(L, vl, R, vr, flr, frl, b.b, part.label)
        assert np.array_equal(F.valid, OV)
        assert np.abs(F.data - OF).max() <= 1e-6


def test_blend_pair_contracts_and_regions(fs, oracle):
    L, vl, R, vr, part, b, flr, frl = _overlap_case(fs, oracle, 30, 12, 12, False)
    ones = np.ones(part.label.shape, np.uint8)
    F = fs.blend_pair(_img(fs, L, vl), _img(fs, R, vr), fs.FlowField(flr, ones),
                      fs.FlowField(frl, ones), b, part)
    a1 = part.label == 1
    assert np.array_equal(F.data[a1], L[a1])
    bad = flr.copy()
    bad[0, 0, 0] = np.nan
    with pytest.raises(fs.ContractError):
        fs.blend_pair(_img(fs, L, vl), _img(fs, R, vr), fs.FlowField(bad, ones),
                      fs.FlowField(frl, ones), b, part)
    with pytest.raises(fs.ContractError):
        fs.blend_pair(_img(fs, L, vl), _img(fs, R, vr), fs.FlowField(flr, ones),
                      fs.FlowField(frl, ones), b, part, fs.BlendParams(0.0))


def test_feather_and_warp_constituents(fs, oracle):
    L, vl, R, vr, part, b, flr, frl = _overlap_case(fs, oracle, 64, 48, 7)
    ones = np.ones(part.label.shape, np.uint8)
    Fe = fs.feather_blend(_img(fs, L, vl), _img(fs, R, vr), b, part)
    a3 = part.label == 3
    exp = (1 - b.b[..., None]) * L + b.b[..., None] * R
    assert np.abs(Fe.data[a3] - exp[a3]).max() <= 1e-6
    # the oracle restatement of proj/src/blender.cpp:102-135 (itself pinned to
    # the compiled reference, tests/test_oracle.py): bit-exact, valid too
    of, ofv = oracle.feather_blend(L, R, b.b, part.label)
    assert np.array_equal(Fe.data, of) and np.array_equal(Fe.valid, ofv)
    wl, wr = fs.warp_constituents(_img(fs, L, vl), _img(fs, R, vr), fs.FlowField(flr, ones),
                                  fs.FlowField(frl, ones), b, part)
    # proj/src/blender.cpp:137-163: the samples Code 1 blends, bit-exact
    (owl, owlv), (owr, owrv) = oracle.warp_constituents(L, vl, R, vr, flr, frl, b.b, part.label)
    assert np.array_equal(wl.data, owl) and np.array_equal(wl.valid, owlv)
    assert np.array_equal(wr.data, owr) and np.array_equal(wr.valid, owrv)
    F = fs.blend_pair(_img(fs, L, vl), _img(fs, R, vr), fs.FlowField(flr, ones),
                      fs.FlowField(frl, ones), b, part)
    lo = np.minimum(wl.data, wr.data) - 1e-6
    hi = np.maximum(wl.data, wr.data) + 1e-6
    assert np.all(F.data[a3] >= lo[a3]) and np.all(F.data[a3] <= hi[a3])


# ---------------------------------------------------------------- seam metric
def _misalign_cases():
    v = np.ones((120, 160), np.uint8)
    tex = S.value_noise(120, 160, 13).astype(np.float32)
    yield tex, v, tex, v, v, v, 16
    yield tex, v, np.roll(tex, 4, axis=1), v, v, v, 16
    yield tex, v, np.roll(tex, (4, 3), axis=(0, 1)), v, v, v, 16
    rng = np.random.RandomState(5)
    L = _rgb(90, 130, 7)
    R = np.roll(L, (2, -3), axis=(0, 1))
    vl = np.ones((90, 130), np.uint8)
    vl[:, 100:] = 0
    vr = np.ones((90, 130), np.uint8)
    vr[:, :20] = 0
    vr[rng.rand(90, 130) > 0.995] = 0
    yield L, vl, R, vr, vl, vr, 16
    yield L, vl, R, vr, vl, vr, 32  # the reference's default stride


@pytest.mark.parametrize("case", list(range(5)))
def test_misalignment_score_bit_exact(fs, oracle, case):
    L, vl, R, vr, ml, mr, stride = list(_misalign_cases())[case]
    part = fs.compute_partition(fs.Mask(ml), fs.Mask(mr))
    got = fs.misalignment_score(_img(fs, L, vl), _img(fs, R, vr), part, 8, stride)
    exp = oracle.misalignment_score(L, vl, R, vr, part.label, part.counts, 8, stride)
    assert got == exp


def test_misalignment_score_errors_and_seam_reduction(fs, oracle):
    v = np.ones((120, 160), np.uint8)
    flat = np.full((120, 160), 0.2, np.float32)
    part = fs.compute_partition(fs.Mask(v), fs.Mask(v))
    with pytest.raises(fs.EmptyRegionError):  # test_pipeline.cpp:191-194
        fs.misalignment_score(_img(fs, flat), _img(fs, flat), part, 8, 16)
    with pytest.raises(fs.ContractError):
        fs.misalignment_score(_img(fs, flat), _img(fs, flat), part, 0, 16)
    # acceptance.cpp:265-294: warped constituents score far below the raw pair
    L, vl, R, vr, part, b, flr, frl = _overlap_case(fs, oracle, 160, 120, 3)
    ones = np.ones(part.label.shape, np.uint8)
    wl, wr = fs.warp_constituents(_img(fs, L, vl), _img(fs, R, vr), fs.FlowField(flr, ones),
                                  fs.FlowField(frl, ones), b, part)
    before = fs.misalignment_score(_img(fs, L, vl), _img(fs, R, vr), part, 8, 16)
    after = fs.misalignment_score(wl, wr, part, 8, 16)
    assert before == oracle.misalignment_score(L, vl, R, vr, part.label, part.counts, 8, 16)
    assert after == oracle.misalignment_score(wl.data, wl.valid, wr.data, wr.valid, part.label,
                                              part.counts, 8, 16)


def test_estimate_translation_matches_oracle(fs, oracle):
    a = S.value_noise(64, 64, 8).astype(np.float32)
    b = np.roll(a, (-3, 5), axis=(0, 1))
    rng = np.random.RandomState(3)
    c = (a + 0.01 * rng.rand(64, 64)).astype(np.float32)
    d = S.value_noise(96, 150, 2).astype(np.float32)
    e = np.roll(d, (7, -11), axis=(0, 1))
    for A, B, m in ((a, b, 8), (a, a, 4), (a, c, 6), (b, a, 16), (d, e, 20)):
        t = fs.estimate_translation(_img(fs, A), _img(fs, B), m)
        assert (t.dx, t.dy, t.score) == oracle.estimate_translation(A, B, m)
    t = fs.estimate_translation(_img(fs, a), _img(fs, b), 8)  # test_pipeline.cpp:151-158
    assert (t.dx, t.dy) == (5, -3) and t.score > 0.99
    flat = np.full((64, 64), 0.5, np.float32)
    with pytest.raises(fs.EmptyRegionError):
        fs.estimate_translation(_img(fs, flat), _img(fs, flat), 4)
    with pytest.raises(fs.ContractError):
        fs.estimate_translation(_img(fs, a), _img(fs, a), 40)
    with pytest.raises(fs.ContractError):
        fs.estimate_translation(_img(fs, _rgb(64, 64, 1)), _img(fs, _rgb(64, 64, 1)), 4)


# ---------------------------------------------------------------- fold
def _fold_both(fs, oracle, lay, params):
    fv = lay.float_views()
    placed = [fs.PlacedImage(fs.ImageBuf(d, v), x, y) for (d, v), (x, y) in zip(fv, lay.offsets)]
    pano, rep = fs.stitch_placed(placed, lay.canvas_w, lay.canvas_h, params)
    od, ov = oracle.stitch_placed([d for d, _ in fv], [v for _, v in fv], lay.offsets,
                                  lay.canvas_w, lay.canvas_h, params.astuple())
    return pano, rep, od, ov


@pytest.mark.parametrize("builder,kw", [(S.small_strip, dict(levels=3, window_radius=5,
                                                               iterations_per_level=2)),
                                        (S.small_panorama, dict(levels=3))])
def test_stitch_placed_matches_oracle(fs, oracle, builder, kw):
    lay = builder(seed=3)
    pano, rep, od, ov = _fold_both(fs, oracle, lay, fs.FlowParams(**kw))
    assert np.array_equal(pano.valid, ov)
    assert np.abs(pano.data - od).max() <= 1e-5
    assert len(rep.pairs) == len(lay.views) - 1
    q_gpu = np.rint(np.clip(pano.data, 0, 1) * 255)
    q_ref = np.rint(np.clip(od, 0, 1) * 255)
    assert np.mean(np.abs(q_gpu - q_ref) <= 1) >= 0.999


@pytest.mark.parametrize("builder", [S.small_strip, S.small_panorama])
def test_stitch_report_seam_metrics_match_reference(fs, ref, builder):
    """StitchReport.pairs[k].misalignment_before / after (pipeline.cpp:184-199)
    against the compiled reference's own report.  The first pair's raw metric
    reads only view 0 and view 1: bit-identical.  The others see panoramas
    and warps built from flows that agree to ~1e-5 px: the best integer
    shifts, hence the scores, agree (checked to 1e-9)."""
    lay = builder(seed=3)
    params = fs.FlowParams(levels=3)
    fv = lay.float_views()
    placed = [fs.PlacedImage(fs.ImageBuf(d, v), x, y) for (d, v), (x, y) in zip(fv, lay.offsets)]
    pano, rep = fs.stitch_placed(placed, lay.canvas_w, lay.canvas_h, params)
    ref.stitch_placed([d for d, _ in fv], [v for _, v in fv], lay.offsets, lay.canvas_w,
                      lay.canvas_h, params.astuple(), full=True)
    exp = ref.last_report_misalignment()
    assert len(exp) == len(rep.pairs)
    got = np.array([[np.nan if p.misalignment_before is None else p.misalignment_before,
                     np.nan if p.misalignment_after is None else p.misalignment_after]
                    for p in rep.pairs])
    assert np.array_equal(np.isnan(got), np.isnan(exp))
    assert got[0, 0] == exp[0, 0]
    ok = ~np.isnan(exp)
    assert np.abs(got[ok] - exp[ok]).max() <= 1e-9, (got, exp)


def test_stitch_errors(fs):
    img = fs.ImageBuf(_rgb(40, 40, 2), np.ones((40, 40), np.uint8))
    with pytest.raises(fs.EmptyRegionError):
        fs.stitch_placed([fs.PlacedImage(img, 0, 0), fs.PlacedImage(img, 100, 0)], 200, 40)
    with pytest.raises(fs.ContractError):
        fs.stitch_placed([fs.PlacedImage(img, 0, 0)], 200, 40)
    with pytest.raises(fs.LayoutError):
        fs.stitch_placed([fs.PlacedImage(img, 0, 0), fs.PlacedImage(img, 170, 0)], 200, 40)


def test_identity_stitch(fs):
    # test_pipeline.cpp:84-94: two identical placements reproduce the input
    d = _rgb(60, 80, 5)
    img = fs.ImageBuf(d, np.ones((60, 80), np.uint8))
    pano, rep = fs.stitch_placed([fs.PlacedImage(img, 0, 0), fs.PlacedImage(img, 0, 0)], 80, 60,
                                 fs.FlowParams(levels=3, window_radius=5, iterations_per_level=2))
    assert rep.pairs[0].overlap_pixels == 80 * 60
    assert np.allclose(pano.data, d, rtol=1e-4, atol=1e-6)


def test_plan_matches_oracle(fs, oracle):
    lay = S.small_panorama(seed=5)
    params = fs.FlowParams(levels=3)
    fv = lay.float_views()
    od, ov = oracle.stitch_placed([d for d, _ in fv], [v for _, v in fv], lay.offsets,
                                  lay.canvas_w, lay.canvas_h, params.astuple())
    plan = fs.Plan(lay.dims, lay.offsets, lay.canvas_w, lay.canvas_h, params)
    out = np.empty((lay.canvas_h, lay.canvas_w, 4), np.uint8)
    plan.execute_host(lay.views, out)
    assert np.array_equal(out[..., 3] == 255, ov == 1)
    q = np.rint(np.clip(od, 0, 1) * 255).astype(np.int32)
    diff = np.abs(out[..., :3].astype(np.int32) - q)[ov == 1]
    assert diff.max() <= 1 and np.mean(diff == 0) >= 0.999
    # masks given at plan time produce the same boxes
    plan2 = fs.Plan(lay.dims, lay.offsets, lay.canvas_w, lay.canvas_h, params,
                    views_rgba=lay.views)
    for k in range(1, len(lay.views)):
        assert plan.fold_info(k) == plan2.fold_info(k)
    out2 = np.empty_like(out)
    plan.execute_host(lay.views, out2)
    assert np.array_equal(out, out2), "replay is not deterministic"
    plan.close()
    plan2.close()


def test_plan_serial_schedule_many_views(fs, oracle):
    """More views than the DAG schedule takes (kMaxDagViews = 16): the plan
    folds serially on one stream; same panorama as the restatement."""
    lay = S.small_strip(seed=6, n=18, vw=90, vh=72, step=60, parallax=2)
    params = fs.FlowParams(levels=2, window_radius=4, iterations_per_level=2)
    fv = lay.float_views()
    od, ov = oracle.stitch_placed([d for d, _ in fv], [v for _, v in fv], lay.offsets,
                                  lay.canvas_w, lay.canvas_h, params.astuple())
    plan = fs.Plan(lay.dims, lay.offsets, lay.canvas_w, lay.canvas_h, params)
    out = np.empty((lay.canvas_h, lay.canvas_w, 4), np.uint8)
    plan.execute_host(lay.views, out)
    assert np.array_equal(out[..., 3] == 255, ov == 1)
    q = np.rint(np.clip(od, 0, 1) * 255).astype(np.int32)
    diff = np.abs(out[..., :3].astype(np.int32) - q)[ov == 1]
    assert diff.max() <= 1 and np.mean(diff == 0) >= 0.999
    with pytest.raises(fs.FlowstitchError):
        plan.timeline()  # the diagnostics need the DAG schedule
    plan.close()


def _random_layout(seed):
    """A random fold: 2-6 views of random sizes placed so that each overlaps
    the union of the earlier ones, some with alpha holes; random canvas."""
    rng = np.random.RandomState(seed)
    W, H = int(rng.randint(220, 420)), int(rng.randint(140, 300))
    scene = S.rgb_scene(H, W, seed + 100)
    n = int(rng.randint(2, 7))
    offs, views = [], []
    covered = np.zeros((H, W), bool)
    for k in range(n):
        for _ in range(100):
            w, h = int(rng.randint(60, W // 2 + 60)), int(rng.randint(50, H))
            w, h = min(w, W), min(h, H)
            x, y = int(rng.randint(0, W - w + 1)), int(rng.randint(0, H - h + 1))
            if k == 0 or covered[y:y + h, x:x + w].sum() >= 400:
                break
        else:
            break
        v = S.rgba(np.roll(scene, (int(rng.randint(-2, 3)), int(rng.randint(-3, 4))),
                           axis=(0, 1))[y:y + h, x:x + w])
        if rng.rand() < 0.4:  # an alpha hole
            hx, hy = int(rng.randint(0, w)), int(rng.randint(0, h))
            v[hy:hy + int(rng.randint(3, 30)), hx:hx + int(rng.randint(3, 30)), 3] = 0
        valid = v[..., 3] >= 128
        if k > 0 and (covered[y:y + h, x:x + w] & valid).sum() == 0:
            break
        covered[y:y + h, x:x + w] |= valid
        views.append(v)
        offs.append((x, y))
    return S.Layout("random%d" % seed, W, H, views, offs, 3)


@pytest.mark.parametrize("seed", list(range(20)))
def test_plan_random_layouts(fs, oracle, seed):
    """Random layouts through the planned DAG (owner plane, early Area2
    copies, hybrid crops, split read-backs): the planned 8-bit canvas equals
    the device fold's panorama quantised, and the fold matches the
    restatement."""
    lay = _random_layout(seed)
    if len(lay.views) < 2:
        pytest.skip("degenerate layout")
    params = fs.FlowParams(levels=2, window_radius=4, iterations_per_level=2)
    fv = lay.float_views()
    od, ov = oracle.stitch_placed([d for d, _ in fv], [v for _, v in fv], lay.offsets,
                                  lay.canvas_w, lay.canvas_h, params.astuple())
    placed = [fs.PlacedImage(fs.ImageBuf(d, v), x, y) for (d, v), (x, y) in zip(fv, lay.offsets)]
    pano, _ = fs.stitch_placed(placed, lay.canvas_w, lay.canvas_h, params)
    assert np.array_equal(pano.valid, ov)
    assert np.abs(pano.data - od).max() <= 1e-4
    v32 = np.clip(pano.data, 0, 1).astype(np.float32) * np.float32(255.0)
    q_dev = np.floor(v32.astype(np.float64) + 0.5).astype(np.int32)
    plan = fs.Plan(lay.dims, lay.offsets, lay.canvas_w, lay.canvas_h, params,
                   views_rgba=lay.views)
    import torch
    pin = [torch.from_numpy(v).pin_memory() for v in lay.views]
    out = torch.zeros((lay.canvas_h, lay.canvas_w, 4), dtype=torch.uint8).pin_memory()
    for _ in range(2):  # page-locked: the graph with the transfers inside
        plan.execute_ptrs([t.data_ptr() for t in pin], out.data_ptr())
        o = out.numpy()
        assert np.array_equal(o[..., 3] == 255, ov == 1)
        assert np.array_equal(o[..., :3].astype(np.int32)[ov == 1], q_dev[ov == 1])
    plan.close()


def _far_seed_layout(seed=8):
    """Area3 (x 3..500) whose only Area1 seeds are a 3-px hole at its left
    end, while the panorama's bounding box (view 0's rectangle, alpha 0 for
    x >= 500) reaches x = 1000: the bounded distance-transform domain is
    clipped on the right and its exactness certificate fails, so the fold
    must fall back to the full domain."""
    W, H = 1000, 40
    scene = S.rgb_scene(H, W, seed)
    v0 = S.rgba(scene[:, :1000])
    v0[:, 500:, 3] = 0
    v1 = S.rgba(np.roll(scene, 2, axis=1)[:, :500])
    v1[:, :3, 3] = 0
    return S.Layout("far-seed", W, H, [v0, v1], [(0, 0), (0, 0)], 2)


def test_edt_certificate_fallback(fs, oracle):
    lay = _far_seed_layout()
    params = fs.FlowParams(levels=2, window_radius=4, iterations_per_level=2)
    fv = lay.float_views()
    od, ov = oracle.stitch_placed([d for d, _ in fv], [v for _, v in fv], lay.offsets,
                                  lay.canvas_w, lay.canvas_h, params.astuple())
    # device fold (re-runs the fold's transforms on the full domain at once)
    placed = [fs.PlacedImage(fs.ImageBuf(d, v), x, y) for (d, v), (x, y) in zip(fv, lay.offsets)]
    pano, _ = fs.stitch_placed(placed, lay.canvas_w, lay.canvas_h, params)
    assert np.array_equal(pano.valid, ov)
    assert np.abs(pano.data - od).max() <= 1e-5
    # planned fold: the check widens the plan and execute_host runs again;
    # same kernels as the device fold, so its 8-bit canvas is that fold's
    # panorama quantised (src/image.cpp:60-61: lroundf(v * 255.0f))
    plan = fs.Plan(lay.dims, lay.offsets, lay.canvas_w, lay.canvas_h, params,
                   views_rgba=lay.views)
    import torch
    plan.execute(0)
    torch.cuda.synchronize()
    with pytest.raises(fs.ContractError, match="widened"):  # the certificate failed
        plan.check()
    plan.execute(0)
    torch.cuda.synchronize()
    plan.check()  # the widened plan is exact
    out = np.empty((lay.canvas_h, lay.canvas_w, 4), np.uint8)
    v32 = np.clip(pano.data, 0, 1).astype(np.float32) * np.float32(255.0)
    q_dev = np.floor(v32.astype(np.float64) + 0.5).astype(np.int32)
    q_ref = np.rint(np.clip(od, 0, 1) * 255).astype(np.int32)
    for _ in range(2):
        plan.execute_host(lay.views, out)
        assert np.array_equal(out[..., 3] == 255, ov == 1)
        assert np.array_equal(out[..., :3].astype(np.int32)[ov == 1], q_dev[ov == 1])
        assert np.abs(out[..., :3].astype(np.int32) - q_ref)[ov == 1].max() <= 1
    plan.close()


def _skip_wait_layout(seed=4):
    """Fold 3's Area3 box meets fold 1's box but not fold 2's, while fold 2
    writes Area2 pixels inside fold 3's box (view 2's alpha hides its left
    part except a bottom tab): the DAG crops fold 3's L right after compose 1,
    concurrently with fold 2, from the canvas where blended and from the first
    covering view elsewhere."""
    W, H = 600, 400
    scene = S.rgb_scene(H, W, seed)
    rects = [(0, 0, 100, 400), (50, 0, 200, 100), (0, 150, 600, 200), (60, 60, 440, 140)]
    views = []
    for x, y, w, h in rects:
        views.append(S.rgba(scene[y:y + h, x:x + w]))
    a2 = views[2][..., 3]
    a2[:150, :100] = 0  # view 2 meets view 0 only at rows 300-350 (canvas)
    return S.Layout("skip-wait", W, H, views, [(x, y) for x, y, _, _ in rects], 3)


def test_plan_crop_waits_for_last_meeting_box(fs, oracle):
    lay = _skip_wait_layout()
    params = fs.FlowParams(levels=3)
    plan = fs.Plan(lay.dims, lay.offsets, lay.canvas_w, lay.canvas_h, params,
                   views_rgba=lay.views)
    b1, b2, b3 = (plan.fold_info(k)[0] for k in (1, 2, 3))

    def meets(a, b):
        return (min(a[0] + a[2], b[0] + b[2]) > max(a[0], b[0]) and
                min(a[1] + a[3], b[1] + b[3]) > max(a[1], b[1]))
    assert meets(b3, b1) and not meets(b3, b2), (b1, b2, b3)
    fv = lay.float_views()
    od, ov = oracle.stitch_placed([d for d, _ in fv], [v for _, v in fv], lay.offsets,
                                  lay.canvas_w, lay.canvas_h, params.astuple())
    out = np.empty((lay.canvas_h, lay.canvas_w, 4), np.uint8)
    for _ in range(2):
        plan.execute_host(lay.views, out)
        assert np.array_equal(out[..., 3] == 255, ov == 1)
        q = np.rint(np.clip(od, 0, 1) * 255).astype(np.int32)
        diff = np.abs(out[..., :3].astype(np.int32) - q)[ov == 1]
        assert diff.max() <= 1 and np.mean(diff == 0) >= 0.999
    tl = plan.timeline()  # the schedule diagnostics run on this layout too
    assert tl["end"] >= tl["fold3_compose_end"] >= tl["fold3_flow_start"] > 0
    # inside the production graph: a stamp at every LK level of every fold,
    # coarse to fine, between the fold's flow start and its blend
    tg = plan.timeline_graph()
    for k in range(1, plan.n):
        levels = sorted((int(key.rsplit("_L", 1)[1]), t) for key, t in tg.items()
                        if key.startswith("fold%d_L" % k))
        assert levels and levels[0][0] == 0, (k, levels)
        lv = [t for _, t in reversed(levels)]  # coarse to fine
        assert tg["fold%d_flow_start" % k] <= lv[0] and lv == sorted(lv), (k, lv)
        assert lv[-1] <= tg["fold%d_blend_start" % k] <= tg["fold%d_compose_end" % k]
    plan.close()


def _grid_layout(seed=3):
    """2x2 views with a band across the middle: canvas rectangles become
    final after different folds, in both directions."""
    W, H = 420, 300
    scene = S.rgb_scene(H, W, seed)
    offs = [(0, 0), (180, 0), (0, 130), (180, 130), (0, 100)]
    sizes = [(240, 170), (240, 170), (240, 170), (240, 170), (420, 100)]
    views = [S.rgba(scene[y:y + h, x:x + w]) for (x, y), (w, h) in zip(offs, sizes)]
    return S.Layout("grid", W, H, views, offs, 3)


def _gaps_layout(seed=5):
    """A ring-like strip on a taller canvas with a gap column: canvas
    rectangles no view covers (zeroed on the host in the overlap path)."""
    W, H = 520, 260
    scene = S.rgb_scene(H, W, seed)
    offs = [(0, 40), (150, 40), (300, 60), (330, 150)]
    sizes = [(190, 150), (190, 150), (170, 100), (150, 90)]
    views = [S.rgba(np.roll(scene, k, axis=1)[y:y + h, x:x + w])
             for k, ((x, y), (w, h)) in enumerate(zip(offs, sizes))]
    return S.Layout("gaps", W, H, views, offs, 3)


@pytest.mark.parametrize("which", ["panorama", "grid", "gaps"])
def test_plan_host_overlap_matches_sync_path(fs, which):
    """execute_host with page-locked buffers runs the graph whose copies
    overlap the folds (per-view H2D, per-rectangle D2H, uncovered canvas
    zeroed by a host node); it must reproduce the pageable (copy, graph,
    copy) path and the device path."""
    import torch
    lay = {"panorama": lambda: S.small_panorama(seed=2), "grid": _grid_layout,
           "gaps": _gaps_layout}[which]()
    plan = fs.Plan(lay.dims, lay.offsets, lay.canvas_w, lay.canvas_h, fs.FlowParams(levels=3))
    h2d, d2h = plan.transfer_bytes()
    assert h2d == sum(v.nbytes for v in lay.views)
    assert (d2h < lay.canvas_w * lay.canvas_h * 4) == (which == "gaps")
    ref = np.empty((lay.canvas_h, lay.canvas_w, 4), np.uint8)
    plan.execute_host(lay.views, ref)  # pageable numpy: synchronous copies
    pin = [torch.from_numpy(v).pin_memory() for v in lay.views]
    out = torch.full((lay.canvas_h, lay.canvas_w, 4), 7, dtype=torch.uint8).pin_memory()
    for _ in range(2):  # capture, then replay
        out.fill_(7)
        plan.execute_ptrs([t.data_ptr() for t in pin], out.data_ptr())
        assert np.array_equal(out.numpy(), ref)
    # new host buffers: the graph is re-captured for the new pointers
    pin2 = [t.clone().pin_memory() for t in pin]
    out2 = torch.zeros_like(out).pin_memory()
    plan.execute_ptrs([t.data_ptr() for t in pin2], out2.data_ptr())
    assert np.array_equal(out2.numpy(), ref)
    # device-resident execution reads the same panorama from the output buffer
    plan.execute(0)
    torch.cuda.synchronize()

    class _Dev:
        __cuda_array_interface__ = {"shape": ref.shape, "typestr": "|u1", "version": 3,
                                    "data": (plan.output_buffer(), False), "strides": None}
    dev = torch.as_tensor(_Dev(), device="cuda").cpu().numpy()
    assert np.array_equal(dev, ref)
    # output only (views already resident): the in-graph read-back alone
    out.fill_(7)
    plan.execute_host(None, out.numpy())
    assert np.array_equal(out.numpy(), ref)
    plan.close()


# ---------------------------------------------------------------- golden vectors (made by the reference)
def test_gpu_matches_golden_vectors(fs):
    import os
    g = np.load(os.path.join(os.path.dirname(__file__), "golden", "golden_v1.npz"))
    p = g["strip_params"]
    params = fs.FlowParams(int(p[0]), int(p[1]), int(p[2]), float(p[3]), int(p[4]))
    placed = [fs.PlacedImage(fs.ImageBuf(g["strip_view%d" % k], g["strip_valid%d" % k]), int(x), int(y))
              for k, (x, y) in enumerate(g["strip_offsets"])]
    cw, ch = (int(v) for v in g["strip_canvas"])
    pano, _ = fs.stitch_placed(placed, cw, ch, params)
    assert np.array_equal(pano.valid, g["strip_out_valid"])
    assert np.abs(pano.data - g["strip_out"]).max() <= 1e-5
    f = fs.dense_pyr_lk(_img(fs, g["lk_from"]), _img(fs, g["lk_to"]))
    assert np.array_equal(f.valid, g["lk_valid"]) and _epe(f.vec, g["lk_vec"]) <= EPE_TOL
    assert np.array_equal(fs.distance_transform(fs.Mask(g["edt_mask"])).d, g["edt_out"])
    part = fs.RegionPartition(g["bf_label"], g["bf_counts"])
    assert np.array_equal(fs.compute_blend(part).b, g["bf_out"])
    ones = np.ones(g["bp_label"].shape, np.uint8)
    F = fs.blend_pair(_img(fs, g["bp_L"], g["bp_vl"]), _img(fs, g["bp_R"], g["bp_vr"]),
                      fs.FlowField(g["bp_flr"], ones), fs.FlowField(g["bp_frl"], ones),
                      fs.BlendField(g["bp_b"]), fs.RegionPartition(g["bp_label"], np.zeros(4, np.int64)))
    assert np.array_equal(F.valid, g["bp_out_valid"]) and np.abs(F.data - g["bp_out"]).max() <= 1e-6
    pyr = fs.build_pyramid(_img(fs, g["pyr_in"]), 4)
    for k, lv in enumerate(pyr):
        assert np.array_equal(lv.data[..., 0], g["pyr_l%d" % k])


@pytest.mark.parametrize("order", ["crop", "views"])
@pytest.mark.parametrize("which", ["panorama", "gaps", "c2"])
def test_plan_rgb8_host_formats(fs, which, order, monkeypatch):
    """RGB8 host views (alpha implicit) and an RGB8 host canvas give the RGBA8
    path's panorama (its RGB channels), through the overlapped graph
    (page-locked) and the copy / graph / copy path (pageable), with either
    upload order of plan_chunks (the first folds' crop parts first, or whole
    views; FS_UPLOAD_ORDER forces it)."""
    import torch
    monkeypatch.setenv("FS_UPLOAD_ORDER", order)
    lay = {"panorama": lambda: S.small_panorama(seed=2), "gaps": _gaps_layout,
           "c2": lambda: S.c2_panorama(3)}[which]()
    assert all((v[..., 3] == 255).all() for v in lay.views)
    plan = fs.Plan(lay.dims, lay.offsets, lay.canvas_w, lay.canvas_h, fs.FlowParams(levels=3))
    ref = np.empty((lay.canvas_h, lay.canvas_w, 4), np.uint8)
    plan.execute_host(lay.views, ref)
    rgb = [np.ascontiguousarray(v[..., :3]) for v in lay.views]
    for out_ch in (4, 3):
        plan.set_host_format(3, out_ch)
        h2d, d2h = plan.transfer_bytes()
        assert h2d == sum(v.nbytes for v in rgb)
        want = ref if out_ch == 4 else np.ascontiguousarray(ref[..., :3])
        pin = [torch.from_numpy(v).pin_memory() for v in rgb]
        out = torch.full(want.shape, 7, dtype=torch.uint8).pin_memory()
        for _ in range(2):
            out.fill_(7)
            plan.execute_ptrs([t.data_ptr() for t in pin], out.data_ptr())
            assert np.array_equal(out.numpy(), want)
        page = np.full(want.shape, 7, np.uint8)
        plan.execute_host(rgb, page)
        assert np.array_equal(page, want)
    plan.set_host_format(4, 4)
    again = np.empty_like(ref)
    plan.execute_host(lay.views, again)
    assert np.array_equal(again, ref)
    plan.close()


def test_lk_max_radius(fs, oracle):
    """the largest accepted window radius runs every sweep mode
    (ring + staging within the device's 227 KB opt-in, now requested in full:
    r = 48, 215 KB for later iterations); r = 49 is refused up front
    (FS_ERR_UNSUPPORTED -> ContractError), not at launch."""
    h, w = 112, 120
    base = S.value_noise(h + 8, w + 8, seed=45)
    frm, to = base[4:4 + h, 4:4 + w], base[3:3 + h, 6:6 + w]
    p = fs.FlowParams(levels=2, window_radius=48, iterations_per_level=2)
    f = fs.dense_pyr_lk(_img(fs, frm), _img(fs, to), p)
    vec, valid = oracle.dense_pyr_lk(frm, to, p)
    assert np.array_equal(f.valid, valid)
    assert _epe(f.vec, vec) <= EPE_TOL
    with pytest.raises(fs.ContractError, match="maximum"):
        fs.dense_pyr_lk(_img(fs, frm), _img(fs, to), fs.FlowParams(levels=2, window_radius=49))


def test_edt_extent_limit(fs, oracle):
    """squared distances are int32 with a 2^30 - 1 sentinel; the
    widest exact canvas row (32768 px: 32767^2 < 2^30 - 1) matches the
    oracle, one pixel more is refused up front (FS_ERR_UNSUPPORTED)."""
    m = np.zeros((1, 32768), np.uint8)
    m[0, 0] = 1
    d = fs.distance_transform(fs.Mask(m)).d
    assert np.array_equal(d, oracle.distance_transform(m))
    assert d[0, -1] == 32767.0
    with pytest.raises(fs.ContractError, match="exact range"):
        fs.distance_transform(fs.Mask(np.ones((1, 32769), np.uint8)))
