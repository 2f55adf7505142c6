// North_star stage 1: fisheye -> equirectangular
// remap with chromaticity gains.  The reference has no such stage (SPEC.md:12
// leaves pre-processing to Hugin/PanoTools), so its parity is UNPINNED: the
// kernel is checked bit for bit against the numpy restatement in
// oracle/remap.py on the same table.
//
// The table (fisheye source position per canvas pixel) is a per-camera
// constant built once on the host in double; the per-frame work is the
// table-driven bilinear gather, one thread per output pixel, HBM-bound:
// table 8 B + out 4 B + the source taps (~4 B, each source pixel is read
// about once through L1/L2) per pixel.
#include <algorithm>
#include <cmath>
#include <cstring>

#include "fs_engine.cuh"

namespace fs {
namespace {

// byte -> float without the conversion pipe: 2^23 + b as a float's bits
// (exact), minus 2^23; and back for an integer-valued float in [0, 255]
constexpr float kMagic = 8388608.f;

struct RemapTap {
    bool ok;
    size_t p[4];     // tap pixels 00, 10, 01, 11
    float w[4];      // their bilinear weights
};
__device__ __forceinline__ RemapTap remap_tap(float2 m, int sw, int sh) {
    RemapTap t;
    t.ok = m.x >= 0.f && m.y >= 0.f && m.x <= (float)(sw - 1) && m.y <= (float)(sh - 1);
    const float mx = t.ok ? m.x : 0.f, my = t.ok ? m.y : 0.f;
    const int x0 = (int)floorf(mx), y0 = (int)floorf(my);
    const int x1 = min(x0 + 1, sw - 1), y1 = min(y0 + 1, sh - 1);
    const float fx = mx - (float)x0, fy = my - (float)y0;
    t.w[0] = (1.f - fx) * (1.f - fy);
    t.w[1] = fx * (1.f - fy);
    t.w[2] = (1.f - fx) * fy;
    t.w[3] = fx * fy;
    t.p[0] = (size_t)y0 * sw + x0;
    t.p[1] = (size_t)y0 * sw + x1;
    t.p[2] = (size_t)y1 * sw + x0;
    t.p[3] = (size_t)y1 * sw + x1;
    return t;
}
__device__ __forceinline__ unsigned int remap_combine(const RemapTap& t, const float (&v)[4][3],
                                                      const float (&g)[3]) {
    if (!t.ok) return 0u;
    unsigned int packed = 0xFF000000u;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        const float s = ((t.w[0] * v[0][c] + t.w[1] * v[1][c]) + t.w[2] * v[2][c]) + t.w[3] * v[3][c];
        float r = floorf(s * g[c] + 0.5f);
        r = r < 255.f ? r : 255.f;
        packed |= (__float_as_uint(r + kMagic) & 0xFFu) << (8 * c);
    }
    return packed;
}

// Two output pixels per thread (the loads of both issued before either is
// combined).
__global__ void __launch_bounds__(256) k_remap_rgba8(const uint8_t* __restrict__ src, int sw, int sh,
                                                     int channels, const float2* __restrict__ map,
                                                     int w, int h, float g0, float g1, float g2,
                                                     uchar4* __restrict__ out) {
    const int x = 2 * (blockIdx.x * blockDim.x + threadIdx.x);
    const int y = blockIdx.y;
    if (x >= w) return;
    const bool two = x + 1 < w;
    const size_t o = (size_t)y * w + x;
    const float2 ma = map[o];
    const float2 mb = two ? map[o + 1] : make_float2(-1.f, -1.f);
    const RemapTap ta = remap_tap(ma, sw, sh), tb = remap_tap(mb, sw, sh);
    const float g[3] = {g0, g1, g2};
    float va[4][3], vb[4][3];
    if (channels == 4) {  // one 32-bit load per tap
        const unsigned int* s4 = reinterpret_cast<const unsigned int*>(src);
        unsigned int qa[4], qb[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            qa[k] = __ldg(s4 + ta.p[k]);
            qb[k] = __ldg(s4 + tb.p[k]);
        }
#pragma unroll
        for (int k = 0; k < 4; ++k)
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                va[k][c] = __uint_as_float(__byte_perm(qa[k], 0x4B000000u, 0x7440u | c)) - kMagic;
                vb[k][c] = __uint_as_float(__byte_perm(qb[k], 0x4B000000u, 0x7440u | c)) - kMagic;
            }
    } else {
#pragma unroll
        for (int k = 0; k < 4; ++k)
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                va[k][c] = (float)__ldg(src + ta.p[k] * 3 + c);
                vb[k][c] = (float)__ldg(src + tb.p[k] * 3 + c);
            }
    }
    unsigned int* o32 = reinterpret_cast<unsigned int*>(out);
    o32[o] = remap_combine(ta, va, g);
    if (two) o32[o + 1] = remap_combine(tb, vb, g);
}

// Overlap channel sums of view k against the first covering earlier view:
// sums[m][0..2] += view m's channels, sums[m][3..5] += view k's channels.
__global__ void __launch_bounds__(256) k_chroma_sums(const uint8_t* __restrict__ owner, int cw,
                                                     ViewU8 vk, PanoViews pv, int k,
                                                     unsigned long long* __restrict__ sums) {
    __shared__ unsigned long long bins[kMaxDagViews * 6];
    for (int i = threadIdx.x; i < kMaxDagViews * 6; i += blockDim.x) bins[i] = 0;
    __syncthreads();
    const int x = vk.rect.x0 + blockIdx.x * blockDim.x + threadIdx.x;
    // a thread's column mostly meets one earlier view: accumulate in
    // registers, flush to the block's bins when the owner changes
    int cur = -1;
    unsigned int acc[6] = {0, 0, 0, 0, 0, 0};  // <= 8192 rows x 255 per flush fits
    int rows = 0;
    auto flush = [&]() {
        if (cur >= 0)
            for (int i = 0; i < 6; ++i)
                if (acc[i]) atomicAdd(&bins[cur * 6 + i], (unsigned long long)acc[i]);
        for (int i = 0; i < 6; ++i) acc[i] = 0;
        rows = 0;
    };
    for (int y = vk.rect.y0 + blockIdx.y; y < vk.rect.y1() && x < vk.rect.x1(); y += gridDim.y) {
        const uchar4 p = vk.px[(size_t)(y - vk.rect.y0) * vk.rect.w + (x - vk.rect.x0)];
        if (p.w < 128) continue;
        const int m = owner[(size_t)y * cw + x];
        if (m >= k) continue;
        if (m != cur || rows == 8192) {
            flush();
            cur = m;
        }
        const ViewU8& vm = pv.v[m];
        const uchar4 q = vm.px[(size_t)(y - vm.rect.y0) * vm.rect.w + (x - vm.rect.x0)];
        acc[0] += q.x;
        acc[1] += q.y;
        acc[2] += q.z;
        acc[3] += p.x;
        acc[4] += p.y;
        acc[5] += p.z;
        ++rows;
    }
    flush();
    __syncthreads();
    for (int i = threadIdx.x; i < k * 6; i += blockDim.x)
        if (bins[i]) atomicAdd(&sums[i], bins[i]);
}

}  // namespace

namespace launch {
void chroma_sums(const uint8_t* owner, int cw, const ViewU8& vk, const PanoViews& pv, int k,
                 unsigned long long* sums, cudaStream_t s) {
    const int bx = (vk.rect.w + 255) / 256;
    const int by = std::min(vk.rect.h, std::max(1, 148 * 8 / bx));
    k_chroma_sums<<<dim3(bx, by), 256, 0, s>>>(owner, cw, vk, pv, k, sums);
}
void remap_rgba8(const uint8_t* src, int sw, int sh, int channels, const float2* map, int w, int h,
                 const float g[3], uchar4* out, cudaStream_t s) {
    if (w > 0 && h > 0)
        k_remap_rgba8<<<dim3((w + 511) / 512, h), 256, 0, s>>>(src, sw, sh, channels, map, w, h,
                                                               g[0], g[1], g[2], out);
}
}  // namespace launch
}  // namespace fs

using namespace fs;

extern "C" {

fs_status fs_fisheye_map(const fs_fisheye_camera* cam, int canvas_w, int canvas_h, int x0, int y0,
                         int w, int h, float* map_xy) {
    if (!cam || !map_xy || canvas_w <= 0 || canvas_h <= 0 || w < 0 || h < 0) {
        last_error_slot() = "fisheye_map: invalid arguments";
        return FS_ERR_CONTRACT;
    }
    if (cam->width <= 0 || cam->height <= 0 || !(cam->focal > 0.0) || !(cam->radius > 0.0)) {
        last_error_slot() = "fisheye_map: camera needs a positive size, focal length and radius";
        return FS_ERR_CONTRACT;
    }
    const double PI = 3.14159265358979323846;
    // camera-from-world = (Ry(yaw) Rx(pitch) Rz(roll))^T
    const double cy_ = std::cos(cam->yaw), sy_ = std::sin(cam->yaw);
    const double cp = std::cos(cam->pitch), sp = std::sin(cam->pitch);
    const double cr = std::cos(cam->roll), sr = std::sin(cam->roll);
    const double Ry[3][3] = {{cy_, 0, sy_}, {0, 1, 0}, {-sy_, 0, cy_}};
    const double Rx[3][3] = {{1, 0, 0}, {0, cp, -sp}, {0, sp, cp}};
    const double Rz[3][3] = {{cr, -sr, 0}, {sr, cr, 0}, {0, 0, 1}};
    double A[3][3], R[3][3];
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) A[i][j] = Ry[i][0] * Rx[0][j] + Ry[i][1] * Rx[1][j] + Ry[i][2] * Rx[2][j];
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) R[i][j] = A[i][0] * Rz[0][j] + A[i][1] * Rz[1][j] + A[i][2] * Rz[2][j];
    for (int v = 0; v < h; ++v) {
        const double lat = PI / 2 - ((y0 + v) + 0.5) / canvas_h * PI;
        const double cl = std::cos(lat), sl = std::sin(lat);
        for (int u = 0; u < w; ++u) {
            const double lon = ((x0 + u) + 0.5) / canvas_w * (2 * PI) - PI;
            const double d[3] = {cl * std::sin(lon), sl, cl * std::cos(lon)};
            // R^T d
            const double dx = R[0][0] * d[0] + R[1][0] * d[1] + R[2][0] * d[2];
            const double dy = R[0][1] * d[0] + R[1][1] * d[1] + R[2][1] * d[2];
            const double dz = R[0][2] * d[0] + R[1][2] * d[1] + R[2][2] * d[2];
            float* mo = map_xy + 2 * ((size_t)v * w + u);
            mo[0] = mo[1] = -1.f;
            const double theta = std::acos(dz < -1.0 ? -1.0 : (dz > 1.0 ? 1.0 : dz));
            const double r = cam->focal * theta;
            if (r > cam->radius) continue;
            const double rho = std::sqrt(dx * dx + dy * dy);
            const double sx = rho > 0.0 ? cam->cx + r * (dx / rho) : cam->cx;
            const double sy = rho > 0.0 ? cam->cy - r * (dy / rho) : cam->cy;
            if (sx < 0.0 || sy < 0.0 || sx > cam->width - 1 || sy > cam->height - 1) continue;
            mo[0] = (float)sx;
            mo[1] = (float)sy;
        }
    }
    return FS_OK;
}

}  // extern "C"
