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
}  // namespace metrics
}  // namespace fs
