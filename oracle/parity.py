"""TEST INFRASTRUCTURE — parity measures between the B200 fold and the
compiled reference (oracle/_ref) on identical inputs.

Used by tests/test_fullsize.py and by bench.py's cpu_baseline leg (which
reports them as the bench line's ``parity`` key).  Numpy only.

Gates (BASELINE.json north_star):
  * valid masks bit-exact (canvas validity and every fold's flow valid bits);
  * flow: mean end-point error <= 0.05 px, and EPE <= 0.5 px on >= 99.99 %
    of the crop pixels;
  * 8-bit output: within +-1 LSB on >= 99.9 % of the canvas pixels.
"""
from __future__ import annotations

import numpy as np

FLOW_MEAN_EPE_TOL = 0.05
FLOW_EPE_MAX = 0.5
FLOW_FRAC_WITHIN = 0.9999
LSB_FRAC = 0.999


def quantize_ref(data: np.ndarray) -> np.ndarray:
    """save_image's quantisation (proj/src/image.cpp:56-65):
    lround(clamp(v, 0, 1) * 255.0f), the product in float."""
    v = np.clip(data.astype(np.float32), np.float32(0), np.float32(1)) * np.float32(255.0)
    return np.floor(v.astype(np.float64) + 0.5).astype(np.int32)


def compare_canvas(gpu: np.ndarray, ref: np.ndarray, ref_valid: np.ndarray) -> dict:
    """gpu: (h, w, 3|4) uint8 canvas (alpha = valid when 4 channels);
    ref: the reference's float canvas (h, w, 3) + valid (h, w)."""
    q = quantize_ref(ref)
    d = np.abs(gpu[..., :3].astype(np.int32) - q).max(-1)
    out = {"max_lsb": int(d.max()), "frac_le_1lsb": float((d <= 1).mean()),
           "frac_exact": float((d == 0).mean())}
    if gpu.shape[-1] == 4:
        out["valid_equal"] = bool(np.array_equal(gpu[..., 3] >= 128, ref_valid != 0))
    else:  # RGB8 canvas: only produced when the views cover every pixel
        out["valid_equal"] = bool(ref_valid.all())
    return out


def compare_flow(gpu_vec, gpu_valid, ref_vec, ref_valid) -> dict:
    epe = np.sqrt(((gpu_vec.astype(np.float64) - ref_vec) ** 2).sum(-1))
    return {"n": int(epe.size), "valid_mismatch": int((gpu_valid != ref_valid).sum()),
            "mean_epe": float(epe.mean()), "max_epe": float(epe.max()),
            "frac_gt_0p5": float((epe > FLOW_EPE_MAX).mean())}


def merge_flow_stats(stats) -> dict:
    n = sum(s["n"] for s in stats)
    return {"n": n, "valid_mismatch": sum(s["valid_mismatch"] for s in stats),
            "mean_epe": sum(s["mean_epe"] * s["n"] for s in stats) / n,
            "max_epe": max(s["max_epe"] for s in stats),
            "frac_gt_0p5": sum(s["frac_gt_0p5"] * s["n"] for s in stats) / n}


def fold_flow_stats(plan, ref_folds) -> dict:
    """Every fold's LtoR and RtoL crop flow of `plan` (last execution) vs the
    reference's (oracle.Oracle.stitch_placed_flows); boxes must agree."""
    stats = []
    for f in ref_folds:
        k = f["k"]
        box, _ = plan.fold_info(k)
        if tuple(box) != tuple(f["box"]):
            raise AssertionError("fold %d: crop box %s != reference %s" % (k, box, f["box"]))
        (glr, glv), (grl, grv) = plan.fold_flow(k)
        stats.append(compare_flow(glr, glv, *f["lr"]))
        stats.append(compare_flow(grl, grv, *f["rl"]))
    return merge_flow_stats(stats)


def gates(canvas: dict, flow: dict) -> dict:
    """Pass/fail per north_star gate."""
    return {"valid": canvas["valid_equal"] and flow["valid_mismatch"] == 0,
            "flow_mean_epe": flow["mean_epe"] <= FLOW_MEAN_EPE_TOL,
            "flow_epe_0p5": flow["frac_gt_0p5"] <= 1.0 - FLOW_FRAC_WITHIN,
            "lsb": canvas["frac_le_1lsb"] >= LSB_FRAC}
