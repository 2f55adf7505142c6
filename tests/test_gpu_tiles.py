"""Row/column tiles of the folds' flows (fs_plan_set_tiling).

A tiled fold computes each interior's flow as its own crop + pyramid + LK
over the interior grown by the dependency cone, so in exact arithmetic it
equals the untiled flow.  In floating point the two differ only by the
summation order of the fp32 later-iteration window sums (the CTA tiling of a
narrower crop); the level tensors and eigenvalue decisions are double, so:

  * valid bits identical (tiled vs untiled, and vs the oracle);
  * flow: max |tiled - untiled| <= 1e-3 px, mean EPE <= 1e-5 px;
  * 8-bit canvas: +-1 LSB everywhere, and vs the oracle the fold gates.
"""
import numpy as np
import pytest

import fs_synthetic as S

pytestmark = pytest.mark.gpu


def _run(fs, lay, tile_len=0, margin=32):
    plan = fs.Plan(lay.dims, lay.offsets, lay.canvas_w, lay.canvas_h,
                   fs.FlowParams(levels=lay.levels))
    if tile_len:
        plan.set_tiling(tile_len, margin)
    out = np.empty((lay.canvas_h, lay.canvas_w, 4), np.uint8)
    plan.execute_host(lay.views, out)
    flows = {k: plan.fold_flow(k) for k in range(1, len(lay.views))}
    tiles = {k: plan.tiles(k) for k in range(1, len(lay.views))}
    plan.close()
    return out, flows, tiles


@pytest.fixture(scope="module")
def lay():
    return S.tile_panorama(seed=3)


@pytest.fixture(scope="module")
def untiled(fs, lay):
    return _run(fs, lay)


def test_tile_plan_partitions_the_box(fs, lay):
    plan = fs.Plan(lay.dims, lay.offsets, lay.canvas_w, lay.canvas_h,
                   fs.FlowParams(levels=lay.levels))
    plan.set_tiling(700)
    tiled_folds = 0
    for k in range(1, len(lay.views)):
        box, depth = plan.fold_info(k)
        tiles = plan.tiles(k)
        if not tiles:
            continue
        tiled_folds += 1
        axis = 0 if box[2] >= box[3] else 1
        edges = []
        for reg, inter in tiles:
            lo, n = (inter[0], inter[2]) if axis == 0 else (inter[1], inter[3])
            rlo, rn = (reg[0], reg[2]) if axis == 0 else (reg[1], reg[3])
            assert rlo <= lo and lo + n <= rlo + rn          # region holds the interior
            assert lo % (1 << (depth - 1)) == 0               # level-aligned cuts
            assert rlo % (1 << (depth - 1)) == 0
            edges.append((lo, lo + n))
        edges.sort()
        assert edges[0][0] == 0 and edges[-1][1] == (box[2] if axis == 0 else box[3])
        assert all(a[1] == b[0] for a, b in zip(edges, edges[1:]))  # a partition
    assert tiled_folds == 2  # the two 2048-wide bands; the seams are shorter than 700 x 2
    plan.set_tiling(0)
    assert all(plan.tiles(k) == [] for k in range(1, len(lay.views)))
    plan.close()


def test_tiled_matches_untiled(fs, lay, untiled):
    out_u, flows_u, _ = untiled
    out_t, flows_t, tiles = _run(fs, lay, 700)
    assert sum(len(t) for t in tiles.values()) >= 6
    for k in flows_u:
        for (vu, ku), (vt, kt) in zip(flows_u[k], flows_t[k]):
            assert np.array_equal(ku, kt), "valid bits differ in fold %d" % k
            d = np.abs(vu - vt)
            assert d.max() <= 1e-3, (k, float(d.max()))
            assert float(np.sqrt((d ** 2).sum(-1)).mean()) <= 1e-5
    diff = np.abs(out_u.astype(np.int32) - out_t.astype(np.int32))
    assert diff.max() <= 1
    assert np.array_equal(out_u[..., 3], out_t[..., 3])


def test_tiled_matches_oracle(fs, oracle, lay):
    out_t, _, tiles = _run(fs, lay, 700)
    assert any(tiles.values())
    fv = lay.float_views()
    ref, ref_valid = oracle.stitch_placed([d for d, _ in fv], [v for _, v in fv], lay.offsets,
                                          lay.canvas_w, lay.canvas_h,
                                          fs.FlowParams(levels=lay.levels).astuple())
    q = np.clip(np.rint(np.clip(ref, 0, 1) * 255.0), 0, 255).astype(np.int32)
    d = np.abs(out_t[..., :3].astype(np.int32) - q)
    assert np.array_equal(out_t[..., 3] >= 128, ref_valid != 0)
    assert d.max() <= 1 and (d == 0).mean() >= 0.999


def test_tile_certificate_falls_back_untiled(fs, lay, untiled, monkeypatch):
    # the test hook narrows every tile's certified exact pyramid part by
    # 4096 px after planning: every gather is then outside it, the device
    # certificate refuses the tiles, the execution is repeated untiled and
    # equals the untiled plan bit for bit
    out_u, flows_u, _ = untiled
    monkeypatch.setenv("FS_TILE_CERT_SHRINK", "4096")
    out_t, flows_t, tiles = _run(fs, lay, 700)
    assert not any(tiles.values()), "certificate should have refused the tiles"
    assert np.array_equal(out_u, out_t)
    for k in flows_u:
        for (vu, ku), (vt, kt) in zip(flows_u[k], flows_t[k]):
            assert np.array_equal(ku, kt) and np.array_equal(vu, vt)


def test_tiling_contracts(fs, lay):
    plan = fs.Plan(lay.dims, lay.offsets, lay.canvas_w, lay.canvas_h,
                   fs.FlowParams(levels=lay.levels))
    with pytest.raises(fs.ContractError):
        plan.set_tiling(-1)
    plan.set_tiling(100000)  # longer than every box: nothing to cut
    assert all(plan.tiles(k) == [] for k in range(1, len(lay.views)))
    plan.close()
