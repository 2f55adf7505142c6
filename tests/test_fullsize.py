"""Full-size parity at every BASELINE.json config (VERDICT r1 "what's missing" 1).

Each case folds the config's synthetic views through the production plan
(fs_plan_*: the CUDA-graph DAG bench.py times) and through the reference
itself (oracle/_ref, compiled from /root/reference by oracle/Makefile, all
host threads), on identical inputs (fs_synthetic), at default FlowParams
(levels=4, r=8, 3 iterations, eps 1e-4, 2 smoothing passes; C3 levels=6):

  * canvas validity bit-exact, 8-bit canvas within +-1 LSB on >= 99.9 %;
  * every fold's LtoR and RtoL crop flow (the FlowFields the reference's
    stitch_placed computes, src/pipeline.cpp:171-172): valid bits identical,
    mean EPE <= 0.05 px, EPE <= 0.5 px on >= 99.99 % of the crop pixels;
  * the known ground truth of C1 (12 px) and C3 (80 px block) is recovered
    by both (acceptance.cpp:198-219 criterion at config scale).

Reference fold times on a 16-thread host: C1 ~0.5 s, C3 ~1.5 s, C2 ~11 s,
C4 ~60 s.  Marked slow; the driver's `-m gpu` run includes them.
"""
import json
import os

import numpy as np
import pytest

import fs_synthetic as S
from oracle import parity as P

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "gpurun_out")


def _fold_both(fs, ref, lay, params=None):
    ref.set_threads(os.cpu_count() or 1)
    fv = lay.float_views()
    params = params or fs.FlowParams(levels=lay.levels)
    rp, rv, folds, secs = ref.stitch_placed_flows([d for d, _ in fv], [v for _, v in fv],
                                                  lay.offsets, lay.canvas_w, lay.canvas_h,
                                                  params.astuple())
    plan = fs.Plan(lay.dims, lay.offsets, lay.canvas_w, lay.canvas_h, params)
    out = np.empty((lay.canvas_h, lay.canvas_w, 4), np.uint8)
    plan.execute_host(lay.views, out)
    canvas = P.compare_canvas(out, rp, rv)
    flow = P.fold_flow_stats(plan, folds)
    return plan, out, (rp, rv, folds, secs), canvas, flow


def _record(name, canvas, flow, secs):
    rec = {"config": name, "canvas": canvas, "flow": flow, "reference_s": round(secs, 2),
           "gates": P.gates(canvas, flow)}
    print(json.dumps(rec))
    try:
        os.makedirs(OUT, exist_ok=True)
        with open(os.path.join(OUT, "fullsize_parity.jsonl"), "a") as f:
            f.write(json.dumps(rec) + "\n")
    except OSError:
        pass
    return rec


def _assert_gates(canvas, flow):
    assert canvas["valid_equal"], canvas
    assert flow["valid_mismatch"] == 0, flow
    assert flow["mean_epe"] <= P.FLOW_MEAN_EPE_TOL, flow
    assert flow["frac_gt_0p5"] <= 1.0 - P.FLOW_FRAC_WITHIN, flow
    assert canvas["frac_le_1lsb"] >= P.LSB_FRAC, canvas


def _interior_mean(vec, valid, m=16):
    v = vec[m:-m, m:-m]
    ok = valid[m:-m, m:-m] != 0
    return v[ok].mean(0)


def test_c1_fullsize(fs, ref):
    lay = S.c1_pair(seed=0)
    plan, out, (rp, rv, folds, secs), canvas, flow = _fold_both(fs, ref, lay)
    _record("C1", canvas, flow, secs)
    _assert_gates(canvas, flow)
    (glr, glv), (grl, grv) = plan.fold_flow(1)
    # uniform 12-px parallax: LtoR = (-12, 0), RtoL = (+12, 0)
    for vec, valid, truth in ((glr, glv, lay.truth["ltor"]), (grl, grv, lay.truth["rtol"])):
        m = _interior_mean(vec, valid)
        assert abs(m[0] - truth[0]) <= 0.5 and abs(m[1] - truth[1]) <= 0.5, (m, truth)
    plan.close()


def test_c3_fullsize_deep_pyramid(fs, ref):
    lay = S.c3_large_parallax(seed=0)
    assert lay.levels == 6
    plan, out, (rp, rv, folds, secs), canvas, flow = _fold_both(fs, ref, lay)
    _record("C3", canvas, flow, secs)
    _assert_gates(canvas, flow)
    box, depth = plan.fold_info(1)
    assert depth == 6
    (glr, glv), _ = plan.fold_flow(1)
    # the foreground block (canvas x 1224..1823, y 262..761) moves 80 px:
    # LtoR dx = -80 in its interior (crop x = canvas x - box x)
    x0 = 1224 - box[0] + 40
    blk = glr[262 + 40:762 - 40, x0:x0 + 600 - 80 - 40]
    bv = glv[262 + 40:762 - 40, x0:x0 + 600 - 80 - 40] != 0
    med = np.median(blk[bv], axis=0)
    assert abs(med[0] + 80) <= 0.5 and abs(med[1]) <= 0.5, med
    rlr = folds[0]["lr"][0][262 + 40:762 - 40, x0:x0 + 600 - 80 - 40]
    assert np.median(rlr[bv], axis=0)[0] == pytest.approx(med[0], abs=0.05)
    plan.close()


def test_c2_fullsize_panorama(fs, ref):
    lay = S.c2_panorama(seed=0)
    plan, out, (rp, rv, folds, secs), canvas, flow = _fold_both(fs, ref, lay)
    _record("C2", canvas, flow, secs)
    _assert_gates(canvas, flow)
    assert len(folds) == 5
    plan.close()


def test_c4_fullsize_ring(fs, ref):
    lay = S.c4_ring(seed=0)
    plan, out, (rp, rv, folds, secs), canvas, flow = _fold_both(fs, ref, lay)
    _record("C4", canvas, flow, secs)
    _assert_gates(canvas, flow)
    assert len(folds) == 7
    plan.close()
