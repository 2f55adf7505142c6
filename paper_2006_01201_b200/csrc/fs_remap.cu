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

__global__ void __launch_bounds__(256) k_remap_rgba8(const uint8_t* __restrict__ src, int sw, int sh,
                                                     int channels, const float2* __restrict__ map,
                                                     int w, int h, float g0, float g1, float g2,
                                                     uchar4* __restrict__ out) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const int y = blockIdx.y;
    if (x >= w) return;
    const size_t o = (size_t)y * w + x;
    const float2 m = map[o];
    if (!(m.x >= 0.f && m.y >= 0.f && m.x <= (float)(sw - 1) && m.y <= (float)(sh - 1))) {
        out[o] = make_uchar4(0, 0, 0, 0);
        return;
    }
    const int x0 = (int)floorf(m.x), y0 = (int)floorf(m.y);
    const int x1 = min(x0 + 1, sw - 1), y1 = min(y0 + 1, sh - 1);
    const float fx = m.x - (float)x0, fy = m.y - (float)y0;
    const float w00 = (1.f - fx) * (1.f - fy), w10 = fx * (1.f - fy);
    const float w01 = (1.f - fx) * fy, w11 = fx * fy;
    const float g[3] = {g0, g1, g2};
    float t[4][3];  // the four taps' channels
    const size_t p00 = (size_t)y0 * sw + x0, p10 = (size_t)y0 * sw + x1;
    const size_t p01 = (size_t)y1 * sw + x0, p11 = (size_t)y1 * sw + x1;
    if (channels == 4) {  // one 32-bit load per tap
        const uchar4* s4 = reinterpret_cast<const uchar4*>(src);
        const uchar4 a = __ldg(s4 + p00), b = __ldg(s4 + p10), c = __ldg(s4 + p01), d = __ldg(s4 + p11);
        const uchar4 tp[4] = {a, b, c, d};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            t[k][0] = (float)tp[k].x;
            t[k][1] = (float)tp[k].y;
            t[k][2] = (float)tp[k].z;
        }
    } else {
        const size_t pk[4] = {p00, p10, p01, p11};
#pragma unroll
        for (int k = 0; k < 4; ++k)
#pragma unroll
            for (int c = 0; c < 3; ++c) t[k][c] = (float)__ldg(src + pk[k] * 3 + c);
    }
    uint8_t q[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        const float v = ((w00 * t[0][c] + w10 * t[1][c]) + w01 * t[2][c]) + w11 * t[3][c];
        const float r = floorf(v * g[c] + 0.5f);
        q[c] = (uint8_t)(r < 255.f ? r : 255.f);
    }
    out[o] = make_uchar4(q[0], q[1], q[2], 255);
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
        k_remap_rgba8<<<dim3((w + 255) / 256, h), 256, 0, s>>>(src, sw, sh, channels, map, w, h,
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
