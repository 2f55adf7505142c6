"""CPU: pin the oracle restatement (oracle/fs_oracle.c).

  * bit-exact against the golden vectors the REFERENCE produced
    (tests/golden/golden_v1.npz, tests/golden/make_golden.py);
  * bit-exact against the reference compiled here (oracle/_ref) on seeded
    random cases, when it is built;
  * the known-answer / property tests of the reference's own suites
    (proj/tests/test_*.cpp, proj/tests/acceptance.cpp) run on the oracle.
"""
import math
import os
import subprocess

import numpy as np
import pytest

from oracle import ref_available, reference, restatement
import fs_synthetic as S

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "golden_v1.npz")


@pytest.fixture(scope="module")
def gold():
    return np.load(GOLDEN)


@pytest.fixture(scope="module")
def fso():
    return restatement()


# ---------------------------------------------------------------- golden vectors
def test_golden_strip_fold(fso, gold):
    views = [gold["strip_view%d" % k] for k in range(3)]
    valids = [gold["strip_valid%d" % k] for k in range(3)]
    cw, ch = (int(v) for v in gold["strip_canvas"])
    p = gold["strip_params"]
    out, ov = fso.stitch_placed(views, valids, [tuple(o) for o in gold["strip_offsets"]], cw, ch,
                                (int(p[0]), int(p[1]), int(p[2]), float(p[3]), int(p[4])))
    assert np.array_equal(out, gold["strip_out"]) and np.array_equal(ov, gold["strip_out_valid"])


def test_golden_flow(fso, gold):
    vec, val = fso.dense_pyr_lk(gold["lk_from"], gold["lk_to"])
    assert np.array_equal(vec, gold["lk_vec"]) and np.array_equal(val, gold["lk_valid"])


def test_golden_edt_blendfield_blend_pyramid(fso, gold):
    assert np.array_equal(fso.distance_transform(gold["edt_mask"]), gold["edt_out"])
    assert np.array_equal(fso.compute_blend(gold["bf_label"], gold["bf_counts"]), gold["bf_out"])
    F, FV = fso.blend_pair(gold["bp_L"], gold["bp_vl"], gold["bp_R"], gold["bp_vr"],
                           gold["bp_flr"], gold["bp_frl"], gold["bp_b"], gold["bp_label"])
    assert np.array_equal(F, gold["bp_out"]) and np.array_equal(FV, gold["bp_out_valid"])
    pyr = fso.build_pyramid(gold["pyr_in"], 4)
    for k, lv in enumerate(pyr):
        assert np.array_equal(lv, gold["pyr_l%d" % k])


# ---------------------------------------------------------------- vs compiled reference
needs_ref = pytest.mark.skipif(not ref_available(), reason="oracle/_ref not built")


@needs_ref
@pytest.mark.parametrize("seed", [0, 1, 2])
def test_restatement_matches_reference_random(fso, seed):
    ref = reference()
    rng = np.random.RandomState(seed)
    h, w = 30 + seed * 7, 41 + seed * 5
    m = (rng.rand(h, w) < 0.1).astype(np.uint8)
    m[0, 0] = 1
    assert np.array_equal(fso.distance_transform(m), ref.distance_transform(m))
    ml = (rng.rand(h, w) > 0.3).astype(np.uint8)
    mr = (rng.rand(h, w) > 0.3).astype(np.uint8)
    la, ca = fso.compute_partition(ml, mr)
    lb, cb = ref.compute_partition(ml, mr)
    assert np.array_equal(la, lb) and np.array_equal(ca, cb)
    assert np.array_equal(fso.compute_blend(la, ca), ref.compute_blend(lb, cb))
    img = np.stack([S.value_noise(h, w, seed + 3 * c) for c in range(3)], -1)
    assert np.array_equal(fso.to_gray(img), ref.to_gray(img))
    a, b = fso.crop_overlap(img, ml, la, ca), ref.crop_overlap(img, ml, lb, cb)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1]) and a[2] == b[2]
    for x, y in rng.uniform(-3, w + 3, size=(50, 2)):
        assert np.array_equal(fso.bilinear_sample(img, ml, x, y), ref.bilinear_sample(img, ml, x, y))


@needs_ref
@pytest.mark.parametrize("params", [(4, 8, 3, 1e-4, 2), (3, 5, 2, 1e-4, 0), (5, 3, 1, 1e-3, 3)])
def test_restatement_matches_reference_flow(fso, params):
    ref = reference()
    base = S.value_noise(90, 110, 17)
    frm, to = base[5:85, 5:105], base[3:83, 9:109]
    a, b = fso.dense_pyr_lk(frm, to, params), ref.dense_pyr_lk(frm, to, params)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    L = np.stack([S.value_noise(40, 50, c) for c in range(3)], -1)
    R = np.roll(L, 2, axis=1)
    (alr, alv), (arl, arv) = fso.bidirectional_flow(L, R, params)
    (blr, blv), (brl, brv) = ref.bidirectional_flow(L, R, params)
    assert np.array_equal(alr, blr) and np.array_equal(arl, brl)
    assert np.array_equal(alv, blv) and np.array_equal(arv, brv)


@needs_ref
@pytest.mark.parametrize("seed", [0, 1])
def test_restatement_matches_reference_feather_and_warp(fso, seed):
    # proj/src/blender.cpp:102-163 (feather_blend, warp_constituents)
    ref = reference()
    rng = np.random.RandomState(40 + seed)
    h, w = 33, 47
    L = np.stack([S.value_noise(h, w, seed + c) for c in range(3)], -1)
    R = np.stack([S.value_noise(h, w, seed + 9 + c) for c in range(3)], -1)
    vl = (rng.rand(h, w) > 0.2).astype(np.uint8)
    vr = (rng.rand(h, w) > 0.2).astype(np.uint8)
    vl[:, 30:] = 0
    vr[:, :12] = 0
    lab, cnt = ref.compute_partition(vl, vr)
    b = ref.compute_blend(lab, cnt)
    flr = rng.uniform(-5, 5, size=(h, w, 2)).astype(np.float32)
    frl = rng.uniform(-5, 5, size=(h, w, 2)).astype(np.float32)
    fa, fb = fso.feather_blend(L, R, b, lab), ref.feather_blend(L, R, b, lab)
    assert np.array_equal(fa[0], fb[0]) and np.array_equal(fa[1], fb[1])
    wa, wb = (fso.warp_constituents(L, vl, R, vr, flr, frl, b, lab),
              ref.warp_constituents(L, vl, R, vr, flr, frl, b, lab))
    for x, y in zip(wa, wb):
        assert np.array_equal(x[0], y[0]) and np.array_equal(x[1], y[1])


@needs_ref
def test_restatement_matches_reference_fold(fso):
    ref = reference()
    lay = S.small_panorama(seed=2)
    fv = lay.float_views()
    args = ([d for d, _ in fv], [v for _, v in fv], lay.offsets, lay.canvas_w, lay.canvas_h,
            (3, 8, 3, 1e-4, 2))
    a, av = fso.stitch_placed(*args)
    b, bv = ref.stitch_placed(*args)
    assert np.array_equal(a, b) and np.array_equal(av, bv)
    # the metric-free fold equals the reference's own stitch_placed (metrics included)
    c, cv = ref.stitch_placed(*args, full=True)
    assert np.array_equal(b, c) and np.array_equal(bv, cv)


@needs_ref
def test_reference_acceptance_suite():
    exe = os.path.join(os.path.dirname(reference().path), "acceptance")
    if not os.path.exists(exe):
        pytest.skip("acceptance binary not built")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 criterion failure(s)" in r.stdout


# ---------------------------------------------------------------- reference KATs on the oracle
def _brute_edt(m):
    ys, xs = np.nonzero(m)
    jj, ii = np.mgrid[0:m.shape[0], 0:m.shape[1]]
    d = np.full(m.shape, np.inf)
    for y, x in zip(ys, xs):
        d = np.minimum(d, np.hypot(ii - x, jj - y))
    return d


def test_edt_vs_brute_force(fso):
    # acceptance.cpp:178-202 (50 random masks, up to 64x64)
    rng = np.random.RandomState(2024)
    for _ in range(50):
        w, h = 4 + rng.randint(61), 4 + rng.randint(61)
        m = (rng.randint(0, 7, size=(h, w)) == 0).astype(np.uint8)
        if not m.any():
            m[rng.randint(h), rng.randint(w)] = 1
        assert np.abs(fso.distance_transform(m) - _brute_edt(m)).max() < 1e-6
    # test_blend_field.cpp:42-50
    m = np.zeros((8, 8), np.uint8)
    m[0, 0] = 1
    d = fso.distance_transform(m)
    assert d[4, 3] == pytest.approx(5.0) and d[0, 0] == 0.0 and d[0, 7] == pytest.approx(7.0)


def test_blend_field_conformance(fso):
    # acceptance.cpp:206-256
    rng = np.random.RandomState(7)
    done = 0
    while done < 20:
        w, h = 24 + rng.randint(41), 16 + rng.randint(33)
        lx1 = w // 2 + rng.randint(w // 2)
        rx0 = rng.randint(lx1 - 1)
        l = np.zeros((h, w), np.uint8)
        r = np.zeros((h, w), np.uint8)
        l[rng.randint(4):h - rng.randint(4), :lx1 + 1] = 1
        r[rng.randint(4):h - rng.randint(4), rx0:] = 1
        lab, cnt = fso.compute_partition(l, r)
        if cnt[3] == 0 or cnt[1] == 0 or cnt[2] == 0:
            continue
        done += 1
        b = fso.compute_blend(lab, cnt)
        assert np.all(b[lab == 1] == 0.0) and np.all(b[lab == 2] == 1.0)
        assert np.all(b[lab == 0] == 0.5)
        lm, rm = _brute_edt(lab == 1), _brute_edt(lab == 2)
        exp = np.where(lm + rm > 0, lm / np.maximum(lm + rm, 1e-300), 0.5)
        assert np.abs(b[lab == 3] - exp[lab == 3]).max() < 1e-6
    # test_blend_field.cpp:89-96
    l = np.zeros((1, 10), np.uint8)
    r = np.zeros((1, 10), np.uint8)
    l[0, :7] = 1
    r[0, 4:] = 1
    lab, cnt = fso.compute_partition(l, r)
    b = fso.compute_blend(lab, cnt)[0]
    assert list(b[:4]) == [0.0] * 4 and list(b[7:]) == [1.0] * 3
    assert b[4] == pytest.approx(0.25) and b[5] == pytest.approx(0.5) and b[6] == pytest.approx(0.75)


def test_softmax_kats(fso):
    # test_blender.cpp:131-147, 149-183, 234-239
    sl, sr = fso.softmax_weights(0.75, 0.25, 0.0, 0.0, 10.0, 0.37)
    assert sl == pytest.approx(0.99330714907571527, rel=1e-15)
    sl, sr = fso.softmax_weights(1.0, 0.0, 100.0, 0.0, 5000.0, 0.05)
    assert math.isfinite(sl) and sl == pytest.approx(1.0)
    sl, sr = fso.softmax_weights(1.0, 0.0, 0.0, 0.0, 10.0, 0.05)
    assert sr < 5e-5
    sl, sr = fso.softmax_weights(0.5, 0.5, 8.0, 2.0, 10.0, 0.05)
    assert sl > 0.5 > sr


def test_code1_vs_naive(fso):
    # acceptance.cpp:260-324: the optimized blend equals a naive per-pixel restatement
    rng = np.random.RandomState(300)
    h, w = 40, 48
    L = np.stack([S.value_noise(h, w, 100 + c) for c in range(3)], -1)
    R = np.stack([S.value_noise(h, w, 200 + c) for c in range(3)], -1)
    vl = np.ones((h, w), np.uint8)
    vr = np.ones((h, w), np.uint8)
    vl[:, 34:] = 0
    vr[:, :15] = 0
    lab, cnt = fso.compute_partition(vl, vr)
    b = fso.compute_blend(lab, cnt)
    flr = rng.uniform(-8, 8, size=(h, w, 2)).astype(np.float32)
    frl = rng.uniform(-8, 8, size=(h, w, 2)).astype(np.float32)
    F, _ = fso.blend_pair(L, vl, R, vr, flr, frl, b, lab)
    for j in range(h):
        for i in range(w):
            if lab[j, i] != 3:
                continue
            br = b[j, i]
            bl = 1.0 - br
            cl = fso.bilinear_sample(L, vl, i + frl[j, i, 0] * (1.0 - bl), j + frl[j, i, 1] * (1.0 - bl))
            cr = fso.bilinear_sample(R, vr, i + flr[j, i, 0] * (1.0 - br), j + flr[j, i, 1] * (1.0 - br))
            fl = 1.0 + 0.05 * math.hypot(frl[j, i, 0], frl[j, i, 1])
            fr = 1.0 + 0.05 * math.hypot(flr[j, i, 0], flr[j, i, 1])
            el, er = math.exp(10.0 * bl * fl), math.exp(10.0 * br * fr)
            exp = np.clip((cl * el + cr * er) / (el + er), 0, 1).astype(np.float32)
            assert np.abs(F[j, i] - exp).max() < 1e-6


def test_pyramid_kats(fso):
    # test_flow.cpp:54-89
    img = S.value_noise(16, 16, 11)
    pyr = fso.build_pyramid(img, 2)
    k1 = np.array([1, 4, 6, 4, 1], np.float64) / 16
    pad = np.pad(img.astype(np.float64), 2, mode="edge")
    sm = np.zeros((16, 16))
    for dj in range(5):
        for di in range(5):
            sm += k1[dj] * k1[di] * pad[dj:dj + 16, di:di + 16]
    assert np.allclose(pyr[1], sm[::2, ::2], rtol=1e-5)
    const = fso.build_pyramid(np.full((16, 16), 0.5, np.float32), 2)
    assert np.allclose(const[1], 0.5)
    assert len(fso.build_pyramid(S.value_noise(20, 20, 3), 5)) == 2


def test_lk_kats(fso):
    # zero motion (test_flow.cpp:91-102), textureless (:126-137), translation (acceptance.cpp:328-349)
    img = S.value_noise(48, 48, 21)
    vec, _ = fso.dense_pyr_lk(img, img, (3, 5, 3, 1e-4, 2))
    assert np.sqrt((vec ** 2).sum(-1)).max() <= 1e-3
    flat = np.full((32, 32), 0.7, np.float32)
    vec, val = fso.dense_pyr_lk(flat, flat, (2, 8, 3, 1e-4, 2))
    assert np.all(vec == 0) and np.all(val == 0)
    base = S.value_noise(160, 160, 77)
    for tx, ty in [(3, 0), (0, -4), (5, 3)]:
        frm = base[16:144, 16:144]
        to = base[16 - ty:144 - ty, 16 - tx:144 - tx]
        vec, _ = fso.dense_pyr_lk(frm, to)
        err = np.hypot(vec[16:112, 16:112, 0] - tx, vec[16:112, 16:112, 1] - ty).mean()
        assert err <= 0.5


def test_fold_identity_and_coverage(fso):
    # test_pipeline.cpp:84-94, 125-135: identical placements reproduce the input;
    # output coverage is the union of the inputs
    img = np.stack([S.value_noise(30, 40, c) for c in range(3)], -1)
    v = np.ones((30, 40), np.uint8)
    out, ov = fso.stitch_placed([img, img], [v, v], [(0, 0), (0, 0)], 40, 30, (3, 5, 2, 1e-4, 2))
    assert np.allclose(out, img, rtol=1e-4, atol=1e-6) and ov.all()
    a = np.stack([S.value_noise(40, 60, 3 + c) for c in range(3)], -1)
    b = np.stack([S.value_noise(40, 60, 9 + c) for c in range(3)], -1)
    va = np.ones((40, 60), np.uint8)
    out, ov = fso.stitch_placed([a, b], [va, va], [(0, 0), (40, 0)], 120, 50, (3, 5, 2, 1e-4, 2))
    exp = np.zeros((50, 120), np.uint8)
    exp[:40, :100] = 1
    assert np.array_equal(ov, exp)


# ---------------------------------------------------------------- misalignment_score
def _tex(h, w, seed, ch=1):
    if ch == 1:
        return S.value_noise(h, w, seed).astype(np.float32)
    return np.stack([S.value_noise(h, w, seed + d) for d in (0, 101, 202)], -1).astype(np.float32)


def _misalign_cases():
    v = np.ones((120, 160), np.uint8)
    tex = _tex(120, 160, 13)
    yield "identical", tex, v, tex, v, v, v
    yield "shift4", tex, v, np.roll(tex, 4, axis=1), v, v, v
    yield "diag", tex, v, np.roll(tex, (4, 3), axis=(0, 1)), v, v, v
    rng = np.random.RandomState(5)
    L = _tex(90, 130, 7, 3)
    R = np.roll(L, (2, -3), axis=(0, 1))
    vl = np.ones((90, 130), np.uint8)
    vl[:, 100:] = 0
    vr = np.ones((90, 130), np.uint8)
    vr[:, :20] = 0
    vr[rng.rand(90, 130) > 0.995] = 0  # holes disqualify candidates
    yield "rgb_partial", L, vl, R, vr, vl, vr


@pytest.mark.parametrize("case", list(range(4)))
def test_misalignment_restatement_kats_and_reference(fso, case):
    name, L, vl, R, vr, ml, mr = list(_misalign_cases())[case]
    lab, cnt = fso.compute_partition(ml, mr)
    a = fso.misalignment_score(L, vl, R, vr, lab, cnt, 8, 16)
    # test_pipeline.cpp:175-196: identical -> 0, 4 px -> ~4, (3, 4) -> ~5
    expect = {"identical": 0.0, "shift4": 4.0, "diag": 5.0}.get(name)
    if expect is not None:
        assert abs(a - expect) <= (0.0 if expect == 0.0 else 0.5)
    if ref_available():
        assert a == reference().misalignment_score(L, vl, R, vr, lab, cnt, 8, 16)


def test_misalignment_flat_and_contract(fso):
    from oracle.binding import OracleError
    v = np.ones((120, 160), np.uint8)
    flat = np.full((120, 160), 0.2, np.float32)
    lab, cnt = fso.compute_partition(v, v)
    with pytest.raises(OracleError) as e:  # EmptyRegionError
        fso.misalignment_score(flat, v, flat, v, lab, cnt, 8, 16)
    assert e.value.status == 2
    with pytest.raises(OracleError) as e:  # ContractError: stride
        fso.misalignment_score(flat, v, flat, v, lab, cnt, 8, 0)
    assert e.value.status == 1


# ---------------------------------------------------------------- estimate_translation
def test_estimate_translation_kats_and_reference(fso):
    from oracle.binding import OracleError
    a = S.value_noise(64, 64, 8).astype(np.float32)
    b = np.roll(a, (-3, 5), axis=(0, 1))  # b(x + 5, y - 3) = a(x, y)
    got = fso.estimate_translation(a, b, 8)  # test_pipeline.cpp:151-158
    assert got[:2] == (5, -3) and got[2] > 0.99
    same = fso.estimate_translation(a, a, 4)
    assert same[:2] == (0, 0) and abs(same[2] - 1.0) < 1e-12
    with pytest.raises(OracleError) as e:  # constant images: no texture
        fso.estimate_translation(np.full((64, 64), 0.5, np.float32),
                                 np.full((64, 64), 0.5, np.float32), 4)
    assert e.value.status == 2
    with pytest.raises(OracleError) as e:  # max_shift too large
        fso.estimate_translation(a, a, 40)
    assert e.value.status == 1
    if ref_available():
        ref = reference()
        rng = np.random.RandomState(3)
        c = (a + 0.01 * rng.rand(64, 64)).astype(np.float32)
        for A, B, m in ((a, b, 8), (a, a, 4), (a, c, 6), (b, a, 16)):
            assert fso.estimate_translation(A, B, m) == ref.estimate_translation(A, B, m)
