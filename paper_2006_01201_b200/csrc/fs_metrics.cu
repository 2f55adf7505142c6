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
                                                               int h, int rad, int stride,
                                                               int ngx, int* __restrict__ res) {
    extern __shared__ double sm[];
    const int P = 2 * rad + 1, NP = P * P, S = 2 * rad, RS = 2 * S + P, NW = 2 * S + 1;
    const int NC = NW * NW;
    double* lp = sm;             // L patch, row-major
    double* rg = lp + NP;        // R window RS x RS
    double* nc = rg + RS * RS;   // NCC per candidate (< -1.5: not a candidate)
    uint8_t* rvb = reinterpret_cast<uint8_t*>(nc + NC);
    __shared__ double s_mean, s_var;
    const int t = threadIdx.x;
    const int cx = rad + blockIdx.x * stride, cy = rad + blockIdx.y * stride;
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

}  // namespace

namespace metrics {

int misalign_max_radius() { return 20; }

void misalign(const float* l, const float* r, const uint8_t* rvalid, const uint8_t* label, int w,
              int h, int ch, int rad, int stride, int* res, double* out, cudaStream_t s) {
    const int ngx = w - 2 * rad > 0 ? (w - 2 * rad + stride - 1) / stride : 0;
    const int ngy = h - 2 * rad > 0 ? (h - 2 * rad + stride - 1) / stride : 0;
    static bool configured = false;
    using K = decltype(&k_misalign_point<PlainGray, PlainGray, PlainValid, PlainArea3>);
    K k = &k_misalign_point<PlainGray, PlainGray, PlainValid, PlainArea3>;
    if (!configured) {
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)ms_smem(misalign_max_radius()));
        configured = true;
    }
    if (ngx > 0 && ngy > 0)
        k<<<dim3(ngx, ngy), MS_THREADS, ms_smem(rad), s>>>(PlainGray{l, w, ch}, PlainGray{r, w, ch},
                                                            PlainValid{rvalid, w},
                                                            PlainArea3{label, w}, w, h, rad,
                                                            stride, ngx, res);
    k_misalign_total<<<1, 1, 0, s>>>(res, ngx, ngy, out);
}

}  // namespace metrics
}  // namespace fs
