// Launchers of the per-function API kernels (fs_api_kernels.cu).
#pragma once

#include "fs_device.cuh"

namespace fs {
namespace api {
// scratch[0] receives the mean; scratch[1..256] are partials
void mean_magnitude(const float2* vec, size_t n, double* scratch, cudaStream_t s);
void count_nonfinite(const float* v, size_t n, unsigned long long* cnt, cudaStream_t s);
void to_gray(const float* img, int n, int ch, float* out, cudaStream_t s);
void bilinear_batch(const float* img, const uint8_t* valid, int w, int h, int ch,
                    const double* xy, int n, float* out, cudaStream_t s);
void partition_planes(const uint8_t* ml, const uint8_t* mr, int w, int h, uint8_t* label,
                      unsigned long long* counts, int* box, cudaStream_t s);
void label_box(const uint8_t* label, int w, int h, int* box, cudaStream_t s);
void crop(const float* img, const uint8_t* valid, int w, int ch, const uint8_t* label, int bx,
          int by, int bw, int bh, float* out, uint8_t* out_valid, cudaStream_t s);
void place(const float* img, const uint8_t* valid, int w, int h, int ch, int ox, int oy, int cw,
           float* out, uint8_t* out_valid, cudaStream_t s);
void embed(const float2* vec, const uint8_t* valid, int w, int h, int ox, int oy, int cw, int chh,
           float2* out, uint8_t* out_valid, cudaStream_t s);
void magnitude(const float2* vec, size_t n, float* out, cudaStream_t s);
void sqrt_field(const int* dsq, size_t n, double* out, cudaStream_t s);
void count_nonzero(const uint8_t* m, size_t n, unsigned long long* cnt, cudaStream_t s);
void blend_field(const uint8_t* label, size_t n, int have1, int have2, const int* d1,
                 const int* d2, double* b, cudaStream_t s);
void blend_pair(const float* l, const uint8_t* vl, const float* r, const uint8_t* vr, int w, int h,
                int ch, const float2* flr, const float2* frl, const double* b,
                const uint8_t* label, double k, double coef, float* out, uint8_t* out_valid,
                cudaStream_t s);
void feather(const float* l, const float* r, int w, int h, int ch, const double* b,
             const uint8_t* label, float* out, uint8_t* out_valid, cudaStream_t s);
void warp_constituents(const float* l, const uint8_t* vl, const float* r, const uint8_t* vr, int w,
                       int h, int ch, const float2* flr, const float2* frl, const double* b,
                       const uint8_t* label, float* ol, uint8_t* ovl, float* orr, uint8_t* ovr,
                       cudaStream_t s);
void import_view(const float* img, const uint8_t* valid, size_t n, int ch, float4* out,
                 uint8_t* vout, cudaStream_t s);
}  // namespace api
}  // namespace fs
