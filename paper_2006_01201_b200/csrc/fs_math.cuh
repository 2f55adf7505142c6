// Per-pixel arithmetic of the flow+blend path, written once and compiled for
// both the sm_100a kernels and the host-side scalar helpers of the drop-in
// shim.  Every routine reproduces the reference's operation order and types
// (float vs double) so that, compiled without FMA contraction (-fmad=false on
// the device, -ffp-contract=off on the host), results match the reference
// bit for bit.  Citations are to /root/reference/proj.
#pragma once

#include <cmath>
#include <cstdint>
#include <cstring>

#ifdef __CUDACC__
#define FS_HD __host__ __device__ __forceinline__
#else
#define FS_HD inline
#endif

namespace fs {

FS_HD int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }
// std::clamp(v, lo, hi) on doubles: (v < lo) ? lo : (hi < v) ? hi : v
FS_HD double clampd(double v, double lo, double hi) { return v < lo ? lo : (hi < v ? hi : v); }
FS_HD int imin(int a, int b) { return a < b ? a : b; }
FS_HD int imax(int a, int b) { return a < b ? b : a; }

// src/image.cpp:76-77 — Rec.601, float, left-to-right.
FS_HD float gray3(float r, float g, float b) { return 0.299f * r + 0.587f * g + 0.114f * b; }

// src/flow.cpp:31 — the binomial taps as float.
FS_HD float binom_tap(int t) {
    return t == 0 ? 6.f / 16 : ((t == 1 || t == -1) ? 4.f / 16 : 1.f / 16);
}

// src/flow.cpp:100-111 — sample_level's bilinear fractions after the clamp
// (the taps themselves: level_tap_f, fs_lk.cu).
struct LevelTap {
    int x0, y0, x1, y1;
    double fx, fy;
};
FS_HD float level_combine(const LevelTap& t, float v00, float v10, float v01, float v11) {
    return static_cast<float>((1 - t.fx) * (1 - t.fy) * v00 + t.fx * (1 - t.fy) * v10 +
                              (1 - t.fx) * t.fy * v01 + t.fx * t.fy * v11);
}

// src/flow.cpp:150-166 — align-centres coordinate of fine pixel i in the
// coarse grid (sx = coarse/fine), its bilinear corners and its nearest cell.
struct UpTap {
    int x0, y0, x1, y1, xn, yn;
    double fx, fy;
};
FS_HD UpTap up_tap(int i, int j, double sx, double sy, int cw, int ch) {
    double xc = clampd((i + 0.5) * sx - 0.5, 0.0, cw - 1.0);
    double yc = clampd((j + 0.5) * sy - 0.5, 0.0, ch - 1.0);
    UpTap t;
    t.x0 = static_cast<int>(xc);
    t.y0 = static_cast<int>(yc);
    t.x1 = imin(t.x0 + 1, cw - 1);
    t.y1 = imin(t.y0 + 1, ch - 1);
    t.fx = xc - t.x0;
    t.fy = yc - t.y0;
    t.xn = clampi(static_cast<int>(lround(xc)), 0, cw - 1);
    t.yn = clampi(static_cast<int>(lround(yc)), 0, ch - 1);
    return t;
}
FS_HD float up_combine(const UpTap& t, float f00, float f10, float f01, float f11) {
    double l = (1 - t.fx) * (1 - t.fy) * f00 + t.fx * (1 - t.fy) * f10 +
               (1 - t.fx) * t.fy * f01 + t.fx * t.fy * f11;
    return static_cast<float>(2.0 * l);
}

// src/flow.cpp:300-311 — final magnitude cap (and the per-update cap of
// src/flow.cpp:283-287, the same expression).  The square root is taken only
// when the squared norm is within 2% of cap^2: below that sqrtf(s) < cap for
// certain, so the outcome is exactly the reference's test.
FS_HD void final_cap(float cap, float& x, float& y) {
    const float s = x * x + y * y;
    if (!(s > 0.98f * (cap * cap))) return;
    float mag = sqrtf(s);
    if (mag > cap) {
        x *= cap / mag;
        y *= cap / mag;
    }
}

// (float)(acc / n), as the reference rounds it (double division, then float
// conversion).  On the device without the double division: with inv_n =
// RN(1/n), q = acc * inv_n lies within 2.5 double ulps of RN(acc / n), so both
// round to the same float unless q's 29 bits below float precision are within
// 4 of the float rounding midpoint, or q is outside the normal float range
// (zero excepted); those rare cases divide exactly, out of line (a branch, not
// predicated work).
#ifdef __CUDACC__
__device__ __noinline__ inline float div_exact_slow(double acc, double n) {
    return static_cast<float>(acc / n);
}
#endif
FS_HD float div_to_float(double acc, double n, double inv_n) {
#if defined(__CUDA_ARCH__) && !defined(FS_EXACT_DIV)
    const double q = acc * inv_n;
    const unsigned long long b = (unsigned long long)__double_as_longlong(q);
    const unsigned lo = (unsigned)b & 0x1FFFFFFFu;
    const unsigned e = (unsigned)(b >> 52) & 0x7FFu;
    if ((e - 897u <= 253u && lo - (0x10000000u - 4u) > 8u) || (b << 1) == 0)
        return static_cast<float>(q);
    return div_exact_slow(acc, n);
#else
    (void)inv_n;
    return static_cast<float>(acc / n);
#endif
}

// src/flow.cpp:267-291 — the 2x2 structure-tensor solve of one pixel.
// Returns true (and the updated flow) when lambda_min >= threshold, with
// inv_det = 1/det (the level's stored inverse structure tensor needs it).
// The eigenvalue test of the structure tensor (a, b; b, c) and, when it
// passes, 1/det.
FS_HD bool lk_tensor_ok(double a, double b, double c, double eig_thresh, double& inv_det) {
    double tr = a + c;
    double det = a * c - b * b;
    double disc = tr * tr - 4.0 * det;
    if (disc < 0.0) disc = 0.0;  // std::max(0.0, x)
    double lambda_min = 0.5 * (tr - sqrt(disc));
    if (lambda_min < eig_thresh) return false;
    inv_det = 1.0 / det;
    return true;
}

FS_HD bool lk_solve(double a, double b, double c, double bx, double by, double eig_thresh,
                        float flow_cap, float& dx, float& dy, double& inv_det) {
    if (!lk_tensor_ok(a, b, c, eig_thresh, inv_det)) return false;
    const double det = a * c - b * b;
    float ndx = dx + -div_to_float(c * bx - b * by, det, inv_det);
    float ndy = dy + -div_to_float(a * by - b * bx, det, inv_det);
    final_cap(flow_cap, ndx, ndy);  // src/flow.cpp:283-287
    dx = ndx;
    dy = ndy;
    return true;
}


// src/image.cpp:87-97 — clamp-to-edge bilinear corners and weights.
struct BiTap {
    int xs[4], ys[4];
    double ws[4];
};
FS_HD BiTap bi_tap(int w, int h, double x, double y) {
    x = clampd(x, 0.0, static_cast<double>(w - 1));
    y = clampd(y, 0.0, static_cast<double>(h - 1));
    int x0 = static_cast<int>(floor(x));
    int y0 = static_cast<int>(floor(y));
    int x1 = imin(x0 + 1, w - 1);
    int y1 = imin(y0 + 1, h - 1);
    double fx = x - x0, fy = y - y0;
    BiTap t;
    t.xs[0] = x0; t.xs[1] = x1; t.xs[2] = x0; t.xs[3] = x1;
    t.ys[0] = y0; t.ys[1] = y0; t.ys[2] = y1; t.ys[3] = y1;
    t.ws[0] = (1 - fx) * (1 - fy);
    t.ws[1] = fx * (1 - fy);
    t.ws[2] = (1 - fx) * fy;
    t.ws[3] = fx * fy;
    return t;
}

// src/blender.cpp:18-30
FS_HD void softmax_weights(double blend_l, double blend_r, double mag_rtol, double mag_ltor,
                           double k, double coef, double& sl, double& sr) {
    double flow_l = 1.0 + coef * mag_rtol;
    double flow_r = 1.0 + coef * mag_ltor;
    double arg_l = k * blend_l * flow_l;
    double arg_r = k * blend_r * flow_r;
    // std::max, then exp(arg - m): the larger argument gives exp(0) == 1
    // exactly, so only the other exponential is evaluated
    const bool r_max = arg_l < arg_r;
    const double m = r_max ? arg_r : arg_l;
    double el = r_max ? exp(arg_l - m) : 1.0;
    double er = r_max ? 1.0 : exp(arg_r - m);
    sl = el / (el + er);
    sr = er / (el + er);
}

// src/blend_field.cpp:109-128 — Eq. 1 on Area3 from exact squared distances.
FS_HD double eq1_area3(bool have1, bool have2, int32_t d1sq, int32_t d2sq) {
    if (!have1 || !have2) return 0.5;
    double l = sqrt(static_cast<double>(d1sq)), r = sqrt(static_cast<double>(d2sq));
    return (l + r > 0.0) ? l / (l + r) : 0.5;
}

// src/image.cpp:60-61 — 8-bit output quantisation.
FS_HD uint8_t quantize8(float v) {
    v = v < 0.0f ? 0.0f : (1.0f < v ? 1.0f : v);
    return static_cast<uint8_t>(lroundf(v * 255.0f));
}

}  // namespace fs
