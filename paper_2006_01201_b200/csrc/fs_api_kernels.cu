// sm_100a kernels behind the per-function C-ABI (the reference's value-type
// API: interleaved float images, canvas-sized flows and fields).  The fold
// engine uses the fused kernels in fs_kernels.cu; these serve the drop-in
// entry points one call at a time.
#include <algorithm>
#include <climits>

#include "fs_api_kernels.cuh"

namespace fs {

// src/image.cpp:70-83
__global__ void k_to_gray(const float* __restrict__ img, int n, int ch, float* __restrict__ out) {
    size_t k = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= (size_t)n) return;
    out[k] = ch == 3 ? gray3(img[k * 3], img[k * 3 + 1], img[k * 3 + 2]) : img[k];
}

// interleaved image sampler (ImageBuf layout)
struct ImgSampler {
    const float* data;
    const uint8_t* valid;
    int w, ch;
    __device__ __forceinline__ bool valid_at(int x, int y) const {
        return valid[(size_t)y * w + x] != 0;
    }
    __device__ __forceinline__ float4 value_at(int x, int y) const {
        const float* p = data + ((size_t)y * w + x) * ch;
        return ch == 3 ? make_float4(p[0], p[1], p[2], 0.f) : make_float4(p[0], 0.f, 0.f, 0.f);
    }
};

// src/image.cpp:85-113 (same arithmetic as the fold's gathers)
template <class S>
__device__ void sample(const S& s, int W, int H, int ch, double x, double y, float out[3]) {
    BiTap t = bi_tap(W, H, x, y);
    double wsum = 0.0;
    bool v[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        v[k] = s.valid_at(t.xs[k], t.ys[k]);
        if (v[k]) wsum += t.ws[k];
    }
    if (wsum <= 0.0) {
        out[0] = out[1] = out[2] = 0.f;
        return;
    }
    for (int c = 0; c < ch; ++c) {
        double acc = 0.0;
#pragma unroll
        for (int k = 0; k < 4; ++k)
            if (v[k]) {
                float4 p = s.value_at(t.xs[k], t.ys[k]);
                acc += t.ws[k] * (c == 0 ? p.x : (c == 1 ? p.y : p.z));
            }
        out[c] = (float)(acc / wsum);
    }
}

__global__ void k_bilinear_batch(ImgSampler s, int h, const double* __restrict__ xy, int n,
                                 float* __restrict__ out) {
    int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    float o[3];
    sample(s, s.w, h, s.ch, xy[2 * k], xy[2 * k + 1], o);
    for (int c = 0; c < s.ch; ++c) out[(size_t)k * s.ch + c] = o[c];
}

// Rows are grid-strided: gridDim.y is capped at 65535 (rows() below), any
// image height works.
#define FS_FOR_ROWS(j, h) for (int j = blockIdx.y; j < (h); j += gridDim.y)

// src/image.cpp:115-132 (counts) and :140-148 (Area3 box)
__global__ void k_partition_planes(const uint8_t* __restrict__ ml, const uint8_t* __restrict__ mr,
                                   int w, int h, uint8_t* __restrict__ label,
                                   unsigned long long* counts, int* box) {
    int x = blockIdx.x * blockDim.x + threadIdx.x;
    FS_FOR_ROWS(y, h) {
        uint8_t reg = 0;
        bool in = x < w;
        if (in) {
            size_t p = (size_t)y * w + x;
            bool l = ml[p] != 0, r = mr[p] != 0;
            reg = l ? (r ? 3 : 1) : (r ? 2 : 0);
            label[p] = reg;
        }
        for (int v = 0; v < 4; ++v) {
            unsigned m = __ballot_sync(0xffffffffu, in && reg == v);
            if ((threadIdx.x & 31) == 0 && m) atomicAdd(&counts[v], (unsigned long long)__popc(m));
        }
        bool a3 = in && reg == 3;
        int mn = __reduce_min_sync(0xffffffffu, a3 ? x : INT_MAX);
        int mx = __reduce_max_sync(0xffffffffu, a3 ? x : -1);
        if ((threadIdx.x & 31) == 0 && mx >= 0) {
            atomicMin(&box[0], mn);
            atomicMin(&box[1], y);
            atomicMax(&box[2], mx);
            atomicMax(&box[3], y);
        }
    }
}

// Area3 box from a label plane (crop_overlap on a given partition)
__global__ void k_label_box(const uint8_t* __restrict__ label, int w, int h, int* box) {
    int x = blockIdx.x * blockDim.x + threadIdx.x;
    FS_FOR_ROWS(y, h) {
        bool a3 = x < w && label[(size_t)y * w + x] == 3;
        int mn = __reduce_min_sync(0xffffffffu, a3 ? x : INT_MAX);
        int mx = __reduce_max_sync(0xffffffffu, a3 ? x : -1);
        if ((threadIdx.x & 31) == 0 && mx >= 0) {
            atomicMin(&box[0], mn);
            atomicMin(&box[1], y);
            atomicMax(&box[2], mx);
            atomicMax(&box[3], y);
        }
    }
}

// src/image.cpp:150-160
__global__ void k_crop(const float* __restrict__ img, const uint8_t* __restrict__ valid, int w,
                       int ch, const uint8_t* __restrict__ label, int bx, int by, int bw, int bh,
                       float* __restrict__ out, uint8_t* __restrict__ out_valid) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    FS_FOR_ROWS(j, bh) {
        if (i >= bw) return;
        size_t s = (size_t)(j + by) * w + (i + bx), d = (size_t)j * bw + i;
        bool v = valid[s] != 0;
        for (int c = 0; c < ch; ++c) out[d * ch + c] = v ? img[s * ch + c] : 0.f;
        out_valid[d] = (label[s] == 3 && v) ? 1 : 0;
    }
}

// src/image.cpp:169-175 (the canvas was zero-filled / invalidated first)
__global__ void k_place(const float* __restrict__ img, const uint8_t* __restrict__ valid, int w,
                        int h, int ch, int ox, int oy, int cw, float* __restrict__ out,
                        uint8_t* __restrict__ out_valid) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    FS_FOR_ROWS(j, h) {
        if (i >= w) return;
        size_t s = (size_t)j * w + i, d = (size_t)(j + oy) * cw + (i + ox);
        for (int c = 0; c < ch; ++c) out[d * ch + c] = img[s * ch + c];
        out_valid[d] = valid ? valid[s] : 1;
    }
}

// src/flow.cpp:342-355 (canvas pre-filled with zero flow, valid = 1)
__global__ void k_embed(const float2* __restrict__ vec, const uint8_t* __restrict__ valid, int w,
                        int h, int ox, int oy, int cw, float2* __restrict__ out,
                        uint8_t* __restrict__ out_valid) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    FS_FOR_ROWS(j, h) {
        if (i >= w) return;
        size_t s = (size_t)j * w + i, d = (size_t)(j + oy) * cw + (i + ox);
        out[d] = vec[s];
        out_valid[d] = valid[s];
    }
}

__global__ void k_fill_flow(float2* __restrict__ v, uint8_t* __restrict__ ok, size_t n) {
    size_t k = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    v[k] = make_float2(0.f, 0.f);
    ok[k] = 1;
}

// src/flow.cpp:330-340
__global__ void k_magnitude(const float2* __restrict__ v, size_t n, float* __restrict__ out) {
    size_t k = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    float2 f = v[k];
    out[k] = sqrtf(f.x * f.x + f.y * f.y);
}

// src/blend_field.cpp:82 — sqrt of the exact squared distance
__global__ void k_sqrt_field(const int* __restrict__ dsq, size_t n, double* __restrict__ out) {
    size_t k = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    out[k] = sqrt((double)dsq[k]);
}

__global__ void k_count_nonzero(const uint8_t* __restrict__ m, size_t n,
                                unsigned long long* cnt) {
    size_t k = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    bool nz = k < n && m[k] != 0;
    unsigned b = __ballot_sync(0xffffffffu, nz);
    if ((threadIdx.x & 31) == 0 && b) atomicAdd(cnt, (unsigned long long)__popc(b));
}

// src/blend_field.cpp:109-128 over the whole canvas
__global__ void k_blend_field(const uint8_t* __restrict__ label, size_t n, int have1, int have2,
                              const int* __restrict__ d1, const int* __restrict__ d2,
                              double* __restrict__ b) {
    size_t k = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    double v = 0.5;
    switch (label[k]) {
        case 1: v = 0.0; break;
        case 2: v = 1.0; break;
        case 3: v = (have1 && have2) ? eq1_area3(true, true, d1[k], d2[k]) : 0.5; break;
        default: v = 0.5; break;
    }
    b[k] = v;
}

// src/blender.cpp:43-100 on canvas-sized value types
__global__ void k_blend_pair(ImgSampler L, ImgSampler R, int w, int h, int ch,
                             const float2* __restrict__ flr, const float2* __restrict__ frl,
                             const double* __restrict__ b, const uint8_t* __restrict__ label,
                             double k, double coef, float* __restrict__ out,
                             uint8_t* __restrict__ out_valid) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    FS_FOR_ROWS(j, h) {
        if (i >= w) return;
        size_t p = (size_t)j * w + i;
        uint8_t reg = label[p];
        float res[3] = {0.f, 0.f, 0.f};
        uint8_t v = 1;
        if (reg == 1) {
            for (int c = 0; c < ch; ++c) res[c] = L.data[p * ch + c];
        } else if (reg == 2) {
            for (int c = 0; c < ch; ++c) res[c] = R.data[p * ch + c];
        } else if (reg == 3) {
            double blend_r = b[p];
            double blend_l = 1.0 - blend_r;
            float2 rl = frl[p], lr = flr[p];
            float cl[3], cr[3];
            sample(L, w, h, ch, i + rl.x * (1.0 - blend_l), j + rl.y * (1.0 - blend_l), cl);
            sample(R, w, h, ch, i + lr.x * (1.0 - blend_r), j + lr.y * (1.0 - blend_r), cr);
            double mag_rl = sqrt((double)rl.x * rl.x + (double)rl.y * rl.y);
            double mag_lr = sqrt((double)lr.x * lr.x + (double)lr.y * lr.y);
            double sl, sr;
            softmax_weights(blend_l, blend_r, mag_rl, mag_lr, k, coef, sl, sr);
            for (int c = 0; c < ch; ++c) res[c] = (float)clampd(cl[c] * sl + cr[c] * sr, 0.0, 1.0);
        } else {
            v = 0;
        }
        for (int c = 0; c < ch; ++c) out[p * ch + c] = res[c];
        out_valid[p] = v;
    }
}

// src/blender.cpp:102-135
__global__ void k_feather(const float* __restrict__ l, const float* __restrict__ r, int w, int h,
                          int ch,
                          const double* __restrict__ b, const uint8_t* __restrict__ label,
                          float* __restrict__ out, uint8_t* __restrict__ out_valid) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    FS_FOR_ROWS(j, h) {
        if (i >= w) return;
        size_t p = (size_t)j * w + i;
        uint8_t reg = label[p];
        uint8_t v = 1;
        for (int c = 0; c < ch; ++c) {
            float res = 0.f;
            if (reg == 1)
                res = l[p * ch + c];
            else if (reg == 2)
                res = r[p * ch + c];
            else if (reg == 3)
                res = (float)clampd((1.0 - b[p]) * l[p * ch + c] + b[p] * r[p * ch + c], 0.0, 1.0);
            out[p * ch + c] = res;
        }
        if (reg == 0) v = 0;
        out_valid[p] = v;
    }
}

// src/blender.cpp:137-163 (outputs pre-filled with copies of L and R)
__global__ void k_warp_constituents(ImgSampler L, ImgSampler R, int w, int h, int ch,
                                    const float2* __restrict__ flr,
                                    const float2* __restrict__ frl, const double* __restrict__ b,
                                    const uint8_t* __restrict__ label, float* __restrict__ ol,
                                    uint8_t* __restrict__ ovl, float* __restrict__ orr,
                                    uint8_t* __restrict__ ovr) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    FS_FOR_ROWS(j, h) {
        if (i >= w) return;
        size_t p = (size_t)j * w + i;
        if (label[p] != 3) continue;
        double blend_r = b[p];
        double blend_l = 1.0 - blend_r;
        float c[3];
        sample(L, w, h, ch, i + frl[p].x * (1.0 - blend_l), j + frl[p].y * (1.0 - blend_l), c);
        for (int q = 0; q < ch; ++q) ol[p * ch + q] = c[q];
        ovl[p] = 1;
        sample(R, w, h, ch, i + flr[p].x * (1.0 - blend_r), j + flr[p].y * (1.0 - blend_r), c);
        for (int q = 0; q < ch; ++q) orr[p * ch + q] = c[q];
        ovr[p] = 1;
    }
}

// ImageBuf (interleaved ch) -> float4 + valid plane, for the fold's views
__global__ void k_import_view(const float* __restrict__ img, const uint8_t* __restrict__ valid,
                              size_t n, int ch, float4* __restrict__ out,
                              uint8_t* __restrict__ vout) {
    size_t k = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    out[k] = ch == 3 ? make_float4(img[k * 3], img[k * 3 + 1], img[k * 3 + 2], 0.f)
                     : make_float4(img[k], 0.f, 0.f, 0.f);
    vout[k] = valid ? (valid[k] != 0) : 1;
}

// deterministic mean of |flow| (pipeline.cpp:40-45 mean_of(flow_magnitude)):
// fixed per-block partials, then one thread sums the partials in order.
__global__ void k_mag_partial(const float2* __restrict__ v, size_t n, double* __restrict__ part) {
    __shared__ double sh[256];
    double acc = 0.0;
    size_t chunk = (n + gridDim.x - 1) / gridDim.x;
    size_t a = (size_t)blockIdx.x * chunk, b = a + chunk < n ? a + chunk : n;
    for (size_t k = a + threadIdx.x; k < b; k += blockDim.x) {
        float2 f = v[k];
        acc += sqrtf(f.x * f.x + f.y * f.y);
    }
    sh[threadIdx.x] = acc;
    __syncthreads();
    for (int s = blockDim.x / 2; s > 0; s >>= 1) {
        if (threadIdx.x < s) sh[threadIdx.x] += sh[threadIdx.x + s];
        __syncthreads();
    }
    if (threadIdx.x == 0) part[blockIdx.x] = sh[0];
}
__global__ void k_mag_final(const double* __restrict__ part, int np, size_t n, double* out) {
    double acc = 0.0;
    for (int k = 0; k < np; ++k) acc += part[k];
    *out = n ? acc / (double)n : 0.0;
}
__global__ void k_count_nonfinite(const float* __restrict__ v, size_t n, unsigned long long* cnt) {
    size_t k = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    bool bad = k < n && !isfinite(v[k]);
    unsigned b = __ballot_sync(0xffffffffu, bad);
    if ((threadIdx.x & 31) == 0 && b) atomicAdd(cnt, (unsigned long long)__popc(b));
}

// ---------------------------------------------------------------------------
namespace api {

void mean_magnitude(const float2* vec, size_t n, double* scratch /*>=257*/, cudaStream_t s) {
    k_mag_partial<<<256, 256, 0, s>>>(vec, n, scratch + 1);
    k_mag_final<<<1, 1, 0, s>>>(scratch + 1, 256, n, scratch);
}
void count_nonfinite(const float* v, size_t n, unsigned long long* cnt, cudaStream_t s) {
    k_count_nonfinite<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(v, n, cnt);
}

static inline unsigned nblk(size_t n, int b = 256) { return (unsigned)((n + b - 1) / b); }
static inline dim3 rows(int w, int h, int b = 256) {
    return dim3((w + b - 1) / b, (unsigned)std::min(h, 65535));
}

void to_gray(const float* img, int n, int ch, float* out, cudaStream_t s) {
    k_to_gray<<<nblk(n), 256, 0, s>>>(img, n, ch, out);
}
void bilinear_batch(const float* img, const uint8_t* valid, int w, int h, int ch,
                    const double* xy, int n, float* out, cudaStream_t s) {
    k_bilinear_batch<<<nblk(n), 256, 0, s>>>(ImgSampler{img, valid, w, ch}, h, xy, n, out);
}
void partition_planes(const uint8_t* ml, const uint8_t* mr, int w, int h, uint8_t* label,
                      unsigned long long* counts, int* box, cudaStream_t s) {
    k_partition_planes<<<rows(w, h), 256, 0, s>>>(ml, mr, w, h, label, counts, box);
}
void label_box(const uint8_t* label, int w, int h, int* box, cudaStream_t s) {
    k_label_box<<<rows(w, h), 256, 0, s>>>(label, w, h, box);
}
void crop(const float* img, const uint8_t* valid, int w, int ch, const uint8_t* label, int bx,
          int by, int bw, int bh, float* out, uint8_t* out_valid, cudaStream_t s) {
    k_crop<<<rows(bw, bh), 256, 0, s>>>(img, valid, w, ch, label, bx, by, bw, bh, out, out_valid);
}
void place(const float* img, const uint8_t* valid, int w, int h, int ch, int ox, int oy, int cw,
           float* out, uint8_t* out_valid, cudaStream_t s) {
    k_place<<<rows(w, h), 256, 0, s>>>(img, valid, w, h, ch, ox, oy, cw, out, out_valid);
}
void embed(const float2* vec, const uint8_t* valid, int w, int h, int ox, int oy, int cw, int chh,
           float2* out, uint8_t* out_valid, cudaStream_t s) {
    size_t n = (size_t)cw * chh;
    k_fill_flow<<<nblk(n), 256, 0, s>>>(out, out_valid, n);
    k_embed<<<rows(w, h), 256, 0, s>>>(vec, valid, w, h, ox, oy, cw, out, out_valid);
}
void magnitude(const float2* vec, size_t n, float* out, cudaStream_t s) {
    k_magnitude<<<nblk(n), 256, 0, s>>>(vec, n, out);
}
void sqrt_field(const int* dsq, size_t n, double* out, cudaStream_t s) {
    k_sqrt_field<<<nblk(n), 256, 0, s>>>(dsq, n, out);
}
void count_nonzero(const uint8_t* m, size_t n, unsigned long long* cnt, cudaStream_t s) {
    k_count_nonzero<<<nblk(n), 256, 0, s>>>(m, n, cnt);
}
void blend_field(const uint8_t* label, size_t n, int have1, int have2, const int* d1,
                 const int* d2, double* b, cudaStream_t s) {
    k_blend_field<<<nblk(n), 256, 0, s>>>(label, n, have1, have2, d1, d2, b);
}
void blend_pair(const float* l, const uint8_t* vl, const float* r, const uint8_t* vr, int w, int h,
                int ch, const float2* flr, const float2* frl, const double* b,
                const uint8_t* label, double k, double coef, float* out, uint8_t* out_valid,
                cudaStream_t s) {
    k_blend_pair<<<rows(w, h, 128), 128, 0, s>>>(ImgSampler{l, vl, w, ch}, ImgSampler{r, vr, w, ch},
                                                w, h, ch, flr, frl, b, label, k, coef, out,
                                                out_valid);
}
void feather(const float* l, const float* r, int w, int h, int ch, const double* b,
             const uint8_t* label, float* out, uint8_t* out_valid, cudaStream_t s) {
    k_feather<<<rows(w, h), 256, 0, s>>>(l, r, w, h, ch, b, label, out, out_valid);
}
void warp_constituents(const float* l, const uint8_t* vl, const float* r, const uint8_t* vr, int w,
                       int h, int ch, const float2* flr, const float2* frl, const double* b,
                       const uint8_t* label, float* ol, uint8_t* ovl, float* orr, uint8_t* ovr,
                       cudaStream_t s) {
    k_warp_constituents<<<rows(w, h, 128), 128, 0, s>>>(
        ImgSampler{l, vl, w, ch}, ImgSampler{r, vr, w, ch}, w, h, ch, flr, frl, b, label, ol, ovl,
        orr, ovr);
}
void import_view(const float* img, const uint8_t* valid, size_t n, int ch, float4* out,
                 uint8_t* vout, cudaStream_t s) {
    k_import_view<<<nblk(n), 256, 0, s>>>(img, valid, n, ch, out, vout);
}

}  // namespace api
}  // namespace fs
