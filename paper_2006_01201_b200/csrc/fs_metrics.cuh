// Seam metrics of the fold report (fs_metrics.cu).
#pragma once

#include "fs_device.cuh"

namespace fs {
namespace metrics {
int misalign_max_radius();
// res: 3 ints per grid point (scratch); out[0] = score, out[1] = matched
// patches (0: no textured patch, the reference's EmptyRegionError)
void misalign(const float* l, const float* r, const uint8_t* rvalid, const uint8_t* label, int w,
              int h, int ch, int rad, int stride, int* res, double* out, cudaStream_t s);
// Inside the fold (fs_stitch_placed): L = the canvas before the fold, R = the
// placed view, Area3 = both valid (its bounding box `box`).  wgray == nullptr:
// misalignment_before (before the compose); else misalignment_after on the
// warped constituents, whose Area3 gray values (L, R) the blend stored
// box-indexed in wgray (NaN-filled beforehand: NaN marks non-Area3 pixels).
void misalign_fold(const Canvas& cv, const ViewF4& v, const Rect& box, const float2* wgray,
                   int rad, int stride, int* res, double* out, cudaStream_t s);
size_t fold_points(const Rect& box, int rad, int stride);  // res holds 3 ints per point
// estimate_translation: ncc scratch (2m+1)^2 doubles; out = {any, dx, dy, score}
void translation(const float* a, const float* b, int w, int h, int max_shift, double* ncc,
                 double* out, cudaStream_t s);
}  // namespace metrics
}  // namespace fs
