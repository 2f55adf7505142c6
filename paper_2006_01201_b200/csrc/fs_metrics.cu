// misalignment_score (src/pipeline.cpp:309-396) on the device: the seam
// metric of StitchReport (pipeline.hpp:30-38, misalignment_before/after).
//
// One CTA per grid point (cx, cy) = (r + i*stride, r + j*stride): the L patch
// and the R search window (+-2r) are staged in shared memory as the doubles
// the reference sums (gray per src/image.cpp:70-83); every candidate shift is
// one thread, whose patch statistics and covariance run in the reference's
// row-major order (patch_stats / patch_ncc, src/pipeline.cpp:220-245), so the
// NCC values are bit-identical; the winner is then chosen by one thread
// scanning the candidates in the reference's (dy, dx) order with its fixed
// tie-break (better_candidate, src/pipeline.cpp:247-256) — the 1e-12
// tolerance makes the order matter.  A last single-thread kernel sums the
// best shift norms per grid row in column order, then the rows in order.
#include "fs_metrics.cuh"

namespace fs {
namespace {

constexpr int MS_THREADS = 256;

__device__ __forceinline__ bool better_candidate(double score, int dx, int dy, double best_score,
                                                 int best_dx, int best_dy) {
    if (score > best_score + 1e-12) return true;
    if (score < best_score - 1e-12) return false;
    const long long n2 = (long long)dx * dx + (long long)dy * dy;
    const long long b2 = (long long)best_dx * best_dx + (long long)best_dy * best_dy;
    if (n2 != b2) return n2 < b2;
    if (dx != best_dx) return dx < best_dx;
    return dy < best_dy;
}

template <class GL, class GR, class RV, class A3>
__global__ void __launch_bounds__(MS_THREADS) k_misalign_point(GL gl, GR gr, RV rv, A3 a3, int w,
                                                               int h, int rad, int stride, int gx0,
                                                               int gy0, int ngx,
                                                               int* __restrict__ res) {
    extern __shared__ double sm[];
    const int P = 2 * rad + 1, NP = P * P, S = 2 * rad, RS = 2 * S + P, NW = 2 * S + 1;
    const int NC = NW * NW;
    double* lp = sm;             // L patch, row-major
    double* rg = lp + NP;        // R window RS x RS
    double* nc = rg + RS * RS;   // NCC per candidate (< -1.5: not a candidate)
    uint8_t* rvb = reinterpret_cast<uint8_t*>(nc + NC);
    __shared__ double s_mean, s_var;
    const int t = threadIdx.x;
    const int cx = rad + (gx0 + (int)blockIdx.x) * stride, cy = rad + (gy0 + (int)blockIdx.y) * stride;
    int* out = res + 3 * (blockIdx.y * ngx + blockIdx.x);
    // the patch footprint must lie in Area3 (src/pipeline.cpp:367)
    int bad = 0;
    for (int k = t; k < NP; k += MS_THREADS) {
        const int x = cx - rad + k % P, y = cy - rad + k / P;
        if (!a3(x, y)) bad = 1;
        lp[k] = (double)gl(x, y);
    }
    bad = __syncthreads_or(bad);
    if (bad) {
        if (t == 0) out[0] = 0;
        return;
    }
    if (t == 0) {  // patch_stats (src/pipeline.cpp:220-233)
        double sum = 0.0, sum2 = 0.0;
        for (int k = 0; k < NP; ++k) {
            const double v = lp[k];
            sum += v;
            sum2 += v * v;
        }
        const double mean = sum / NP;
        s_mean = mean;
        s_var = sum2 / NP - mean * mean;
    }
    const int wx0 = cx - S - rad, wy0 = cy - S - rad;
    for (int k = t; k < RS * RS; k += MS_THREADS) {
        const int x = wx0 + k % RS, y = wy0 + k / RS;
        const bool inside = x >= 0 && x < w && y >= 0 && y < h;
        rg[k] = inside ? (double)gr(x, y) : 0.0;
        rvb[k] = inside && rv(x, y);
    }
    __syncthreads();
    const double lmean = s_mean, lvar = s_var;
    if (lvar < 1e-4) {  // flat patch (src/pipeline.cpp:369)
        if (t == 0) out[0] = 0;
        return;
    }
    for (int c = t; c < NC; c += MS_THREADS) {
        const int dx = c % NW - S, dy = c / NW - S;
        const int bx = cx + dx, by = cy + dy;
        double v = -3.0;
        if (!(bx - rad < 0 || bx + rad >= w || by - rad < 0 || by + rad >= h)) {
            const int ox = dx + S, oy = dy + S;  // patch origin in the window
            bool ok = true;
            for (int j = 0; j < P && ok; ++j)
                for (int i = 0; i < P; ++i)
                    if (!rvb[(oy + j) * RS + ox + i]) {
                        ok = false;
                        break;
                    }
            if (ok) {
                double sum = 0.0, sum2 = 0.0;
                for (int j = 0; j < P; ++j)
                    for (int i = 0; i < P; ++i) {
                        const double q = rg[(oy + j) * RS + ox + i];
                        sum += q;
                        sum2 += q * q;
                    }
                const double rmean = sum / NP, rvar = sum2 / NP - rmean * rmean;
                if (lvar <= 1e-12 || rvar <= 1e-12) {
                    v = -2.0;
                } else {  // patch_ncc (src/pipeline.cpp:235-245)
                    double cov = 0.0;
                    for (int j = 0; j < P; ++j)
                        for (int i = 0; i < P; ++i)
                            cov += (lp[j * P + i] - lmean) * (rg[(oy + j) * RS + ox + i] - rmean);
                    cov /= NP;
                    v = cov / sqrt(lvar * rvar);
                }
            }
        }
        nc[c] = v;
    }
    __syncthreads();
    if (t == 0) {
        double best = -2.0;
        int bdx = 0, bdy = 0, found = 0;
        for (int c = 0; c < NC; ++c) {
            const double v = nc[c];
            if (v < -1.5) continue;
            found = 1;
            const int dx = c % NW - S, dy = c / NW - S;
            if (better_candidate(v, dx, dy, best, bdx, bdy)) {
                best = v;
                bdx = dx;
                bdy = dy;
            }
        }
        out[0] = found;
        out[1] = bdx;
        out[2] = bdy;
    }
}

// src/pipeline.cpp:387-395: per grid row in column order, then rows in order
__global__ void k_misalign_total(const int* __restrict__ res, int ngx, int ngy, double* out) {
    double total = 0.0;
    long long matched = 0;
    for (int j = 0; j < ngy; ++j) {
        double row_total = 0.0;
        long long row_matched = 0;
        for (int i = 0; i < ngx; ++i) {
            const int* r = res + 3 * (j * ngx + i);
            if (!r[0]) continue;
            row_total += sqrt((double)r[1] * r[1] + (double)r[2] * r[2]);
            ++row_matched;
        }
        total += row_total;
        matched += row_matched;
    }
    out[0] = matched ? total / (double)matched : 0.0;
    out[1] = (double)matched;
}

// estimate_translation (src/pipeline.cpp:261-307): one thread per shift sums
// its overlap in the reference's row-major order; one thread then picks the
// winner in the reference's (dy, dx) order.
__global__ void k_translation_shift(const float* __restrict__ a, const float* __restrict__ b,
                                    int w, int h, int ms, double* __restrict__ ncc) {
    const int nw = 2 * ms + 1;
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= nw * nw) return;
    const int dx = c % nw - ms, dy = c / nw - ms;
    const int x0 = max(0, -dx), x1 = min(w, w - dx);
    const int y0 = max(0, -dy), y1 = min(h, h - dy);
    double v = -3.0;
    if (x1 > x0 && y1 > y0) {
        const long long n = (long long)(x1 - x0) * (y1 - y0);
        double sa = 0, sb = 0, saa = 0, sbb = 0, sab = 0;
        for (int y = y0; y < y1; ++y) {
            const float* ra = a + (size_t)y * w;
            const float* rb = b + (size_t)(y + dy) * w + dx;
            for (int x = x0; x < x1; ++x) {
                const double va = __ldg(ra + x), vb = __ldg(rb + x);
                sa += va;
                sb += vb;
                saa += va * va;
                sbb += vb * vb;
                sab += va * vb;
            }
        }
        const double va = saa / n - (sa / n) * (sa / n);
        const double vb = sbb / n - (sb / n) * (sb / n);
        if (!(va <= 1e-12 || vb <= 1e-12)) v = (sab / n - (sa / n) * (sb / n)) / sqrt(va * vb);
    }
    ncc[c] = v;
}

__global__ void k_translation_pick(const double* __restrict__ ncc, int ms, double* out) {
    const int nw = 2 * ms + 1;
    double best = -2.0;
    int bdx = 0, bdy = 0, any = 0;
    for (int c = 0; c < nw * nw; ++c) {
        const double v = ncc[c];
        if (v < -2.5) continue;
        any = 1;
        const int dx = c % nw - ms, dy = c / nw - ms;
        if (better_candidate(v, dx, dy, best, bdx, bdy)) {
            best = v;
            bdx = dx;
            bdy = dy;
        }
    }
    out[0] = any;
    out[1] = bdx;
    out[2] = bdy;
    out[3] = best;
}

struct PlainGray {
    const float* img;
    int w, ch;
    __device__ __forceinline__ float operator()(int x, int y) const {
        const float* p = img + ((size_t)y * w + x) * ch;
        return ch == 3 ? gray3(p[0], p[1], p[2]) : p[0];
    }
};
struct PlainValid {
    const uint8_t* v;
    int w;
    __device__ __forceinline__ bool operator()(int x, int y) const {
        return v[(size_t)y * w + x] != 0;
    }
};
struct PlainArea3 {
    const uint8_t* label;
    int w;
    __device__ __forceinline__ bool operator()(int x, int y) const {
        return label[(size_t)y * w + x] == 3;
    }
};

size_t ms_smem(int rad) {
    const size_t P = 2 * rad + 1, RS = 6 * rad + 1, NW = 4 * rad + 1;
    return 8 * P * P + 9 * RS * RS + 8 * NW * NW;
}

// ---- sources of the fold's two calls (src/pipeline.cpp:184-199) ----------
// L = the panorama before the fold, R = the placed view (place_on_canvas:
// its data inside its rectangle, 0 outside), partition Area3 = both valid.
__device__ __forceinline__ float gray_of(float4 v, int ch) {
    return ch == 3 ? gray3(v.x, v.y, v.z) : v.x;
}
struct CanvasGray {
    const float4* rgb;
    int w, ch;
    __device__ __forceinline__ float operator()(int x, int y) const {
        return gray_of(rgb[(size_t)y * w + x], ch);
    }
};
struct ViewGray {
    ViewF4 v;
    int ch;
    __device__ __forceinline__ float operator()(int x, int y) const {
        return v.rect.contains(x, y) ? gray_of(v.value_at(x, y), ch) : 0.f;
    }
};
struct ViewValid {
    ViewF4 v;
    __device__ __forceinline__ bool operator()(int x, int y) const { return v.valid_at(x, y); }
};
struct FoldArea3 {
    const uint8_t* pano_valid;
    int w;
    ViewF4 v;
    __device__ __forceinline__ bool operator()(int x, int y) const {
        return pano_valid[(size_t)y * w + x] && v.valid_at(x, y);
    }
};
// warp_constituents (src/blender.cpp:137-163): on Area3 the warped colours
// are the blend's two bilinear samples (their gray stored by k_blend_area3,
// box-indexed); elsewhere the constituents are L and R unchanged.
struct WarpGrayL {
    const float2* wg;
    Rect box;
    __device__ __forceinline__ float operator()(int x, int y) const {
        return box.contains(x, y) ? wg[(size_t)(y - box.y0) * box.w + (x - box.x0)].x : 0.f;
    }
};
// Area3 of the fold read from the warp buffer (NaN-filled before the blend,
// written on Area3 only): valid also after the canvas has been composed.
struct WarpArea3 {
    const float2* wg;
    Rect box;
    __device__ __forceinline__ bool operator()(int x, int y) const {
        if (!box.contains(x, y)) return false;
        const float v = wg[(size_t)(y - box.y0) * box.w + (x - box.x0)].x;
        return v == v;
    }
};
struct WarpGrayR {
    const float2* wg;
    Rect box;
    WarpArea3 a3;
    ViewGray vg;
    __device__ __forceinline__ float operator()(int x, int y) const {
        return a3(x, y) ? wg[(size_t)(y - box.y0) * box.w + (x - box.x0)].y : vg(x, y);
    }
};

template <class GL, class GR, class RV, class A3>
void launch_points(GL gl, GR gr, RV rv, A3 a3, int w, int h, int rad, int stride, int gx0,
                   int gy0, int ngx, int ngy, int* res, cudaStream_t s) {
    auto k = &k_misalign_point<GL, GR, RV, A3>;
    static std::atomic<unsigned long long> configured{0};
    once_per_device(configured, [&](int) {
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)ms_smem(metrics::misalign_max_radius()));
    });
    if (ngx > 0 && ngy > 0)
        k<<<dim3(ngx, ngy), MS_THREADS, ms_smem(rad), s>>>(gl, gr, rv, a3, w, h, rad, stride, gx0,
                                                            gy0, ngx, res);
}

}  // namespace

namespace metrics {

int misalign_max_radius() { return 20; }

void misalign(const float* l, const float* r, const uint8_t* rvalid, const uint8_t* label, int w,
              int h, int ch, int rad, int stride, int* res, double* out, cudaStream_t s) {
    const int ngx = w - 2 * rad > 0 ? (w - 2 * rad + stride - 1) / stride : 0;
    const int ngy = h - 2 * rad > 0 ? (h - 2 * rad + stride - 1) / stride : 0;
    launch_points(PlainGray{l, w, ch}, PlainGray{r, w, ch}, PlainValid{rvalid, w},
                  PlainArea3{label, w}, w, h, rad, stride, 0, 0, ngx, ngy, res, s);
    k_misalign_total<<<1, 1, 0, s>>>(res, ngx, ngy, out);
}

void translation(const float* a, const float* b, int w, int h, int max_shift, double* ncc,
                 double* out, cudaStream_t s) {
    const int nc = (2 * max_shift + 1) * (2 * max_shift + 1);
    k_translation_shift<<<(nc + 127) / 128, 128, 0, s>>>(a, b, w, h, max_shift, ncc);
    k_translation_pick<<<1, 1, 0, s>>>(ncc, max_shift, out);
}

// Grid points whose footprint lies in the Area3 box: the others cannot have
// their footprint in Area3 and add nothing (exact zeros) to the row sums.
void fold_grid(const Rect& box, int rad, int stride, int& gx0, int& gy0, int& ngx, int& ngy) {
    gx0 = (box.x0 + stride - 1) / stride;
    gy0 = (box.y0 + stride - 1) / stride;
    const int gx1 = box.x1() - 1 - 2 * rad >= 0 ? (box.x1() - 1 - 2 * rad) / stride : -1;
    const int gy1 = box.y1() - 1 - 2 * rad >= 0 ? (box.y1() - 1 - 2 * rad) / stride : -1;
    ngx = gx1 >= gx0 ? gx1 - gx0 + 1 : 0;
    ngy = gy1 >= gy0 ? gy1 - gy0 + 1 : 0;
}

void misalign_fold(const Canvas& cv, const ViewF4& v, const Rect& box, const float2* wgray,
                   int rad, int stride, int* res, double* out, cudaStream_t s) {
    int gx0, gy0, ngx, ngy;
    fold_grid(box, rad, stride, gx0, gy0, ngx, ngy);
    const FoldArea3 a3{cv.valid, cv.w, v};
    const ViewGray vg{v, cv.ch};
    if (!wgray)
        launch_points(CanvasGray{cv.rgb, cv.w, cv.ch}, vg, ViewValid{v}, a3, cv.w, cv.h, rad,
                      stride, gx0, gy0, ngx, ngy, res, s);
    else
        launch_points(WarpGrayL{wgray, box}, WarpGrayR{wgray, box, WarpArea3{wgray, box}, vg},
                      ViewValid{v}, WarpArea3{wgray, box}, cv.w, cv.h, rad, stride, gx0, gy0, ngx,
                      ngy, res, s);
    k_misalign_total<<<1, 1, 0, s>>>(res, ngx, ngy, out);
}

size_t fold_points(const Rect& box, int rad, int stride) {
    int gx0, gy0, ngx, ngy;
    fold_grid(box, rad, stride, gx0, gy0, ngx, ngy);
    return (size_t)ngx * ngy;
}

}  // namespace metrics
}  // namespace fs
