// sm_100a kernels of the flow+blend hot path (K0-K8 of SURVEY.md §2.2).
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false ...
// -fmad=false keeps every float/double expression that mirrors the reference
// un-contracted, which is what makes the outputs bit-comparable with the
// reference's Release build (no -march, hence no FMA).
#include <algorithm>
#include <climits>

#include "fs_device.cuh"

namespace fs {

FS_CHECK_TU(kernels)


// ============================================================================
// K0 — placement, partition statistics, crop + gray
// ============================================================================

// src/image.cpp:164-177 (place_on_canvas) for the first view of a fold: the
// canvas valid plane was cleared; the view's pixels and validity are written
// at its offset and its valid pixels counted.
// Rows of a view rectangle are covered by 256-thread blocks that each walk
// PART_ROWS rows; per-block results are reduced in shared memory so each
// block issues one atomic per statistic (thousands, not millions).
constexpr int PART_ROWS = 8;

// K8 (src/image.cpp:52-65) of one valid pixel: RGBA8, alpha 255
__device__ __forceinline__ uchar4 quantize_px(float4 v, int ch) {
    const uint8_t r = quantize8(v.x);
    return ch == 3 ? make_uchar4(r, quantize8(v.y), quantize8(v.z), 255)
                   : make_uchar4(r, r, r, 255);
}

// out != nullptr (the planned DAG): the RGBA8 canvas is written by each
// pixel's writers directly (place, Area2 copy, Area3 compose) — the last
// writer of a pixel leaves its final 8-bit value.
template <class V>
__global__ void __launch_bounds__(256) k_place_view(Canvas cv, V view, CanvasCount* count,
                                                    uchar4* __restrict__ out, int write_cv) {
    __shared__ int red[8];
    const int x = view.rect.x0 + blockIdx.x * blockDim.x + threadIdx.x;
    const int ya = view.rect.y0 + blockIdx.y * PART_ROWS;
    const int yb = min(ya + PART_ROWS, view.rect.y1());
    int n = 0;
    if (x < view.rect.x1())
        for (int y = ya; y < yb; ++y) {
            size_t p = (size_t)y * cv.w + x;
            bool v = view.valid_at(x, y);
            const float4 val = view.value_at(x, y);
            if (write_cv) {
                cv.rgb[p] = val;
                cv.valid[p] = v ? 1 : 0;
            }
            if (out && v) out[p] = quantize_px(val, cv.ch);
            n += v;
        }
    n = __reduce_add_sync(0xffffffffu, n);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = n;
    __syncthreads();
    if (threadIdx.x == 0) {
        int t = 0;
        for (int k = 0; k < 8; ++k) t += red[k];
        if (t) atomicAdd(&count->valid_count, (unsigned long long)t);
    }
}

// src/image.cpp:115-132 + :140-148, restricted to the view rectangle (Area2 and
// Area3 live there): Area2/Area3 counts and the Area3 bounding box.
template <class V, class P>
__global__ void __launch_bounds__(256) k_partition(P pano, V view, FoldStats* st) {
    __shared__ int red[5][8];
    const int x = view.rect.x0 + blockIdx.x * blockDim.x + threadIdx.x;
    const int ya = view.rect.y0 + blockIdx.y * PART_ROWS;
    const int yb = min(ya + PART_ROWS, view.rect.y1());
    int n2 = 0, n3 = 0, minx = INT_MAX, maxx = -1, miny = INT_MAX, maxy = -1;
    if (x < view.rect.x1()) {
        // the rows' masks loaded first (independent loads), then classified
        bool vv[PART_ROWS], pp[PART_ROWS];
#pragma unroll
        for (int j = 0; j < PART_ROWS; ++j) {
            const int y = ya + j;
            vv[j] = y < yb && view.valid_at(x, y);
            pp[j] = y < yb && pano.valid_at(x, y);
        }
#pragma unroll
        for (int j = 0; j < PART_ROWS; ++j) {
            if (!vv[j]) continue;
            if (pp[j]) {
                ++n3;
                minx = min(minx, x);
                maxx = max(maxx, x);
                miny = min(miny, ya + j);
                maxy = max(maxy, ya + j);
            } else {
                ++n2;
            }
        }
    }
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    n2 = __reduce_add_sync(0xffffffffu, n2);
    n3 = __reduce_add_sync(0xffffffffu, n3);
    minx = __reduce_min_sync(0xffffffffu, minx);
    maxx = __reduce_max_sync(0xffffffffu, maxx);
    miny = __reduce_min_sync(0xffffffffu, miny);
    maxy = __reduce_max_sync(0xffffffffu, maxy);
    if (lane == 0) {
        red[0][wid] = n2;
        red[1][wid] = n3;
        red[2][wid] = minx;
        red[3][wid] = maxx;
        red[4][wid] = (maxy << 0);
    }
    __shared__ int rminy[8];
    if (lane == 0) rminy[wid] = miny;
    __syncthreads();
    if (threadIdx.x == 0) {
        int t2 = 0, t3 = 0, mnx = INT_MAX, mxx = -1, mny = INT_MAX, mxy = -1;
        for (int k = 0; k < 8; ++k) {
            t2 += red[0][k];
            t3 += red[1][k];
            mnx = min(mnx, red[2][k]);
            mxx = max(mxx, red[3][k]);
            mny = min(mny, rminy[k]);
            mxy = max(mxy, red[4][k]);
        }
        if (t2) atomicAdd(&st->cnt2, (unsigned long long)t2);
        if (t3) {
            atomicAdd(&st->cnt3, (unsigned long long)t3);
            atomicMin(&st->bx0, mnx);
            atomicMax(&st->bx1, mxx);
            atomicMin(&st->by0, mny);
            atomicMax(&st->by1, mxy);
        }
    }
}

// Checks the device-measured Area3 box against the planned one.
__global__ void k_check_box(FoldStats* st, Rect planned) {
    bool ok = st->cnt3 > 0 && st->bx0 == planned.x0 && st->by0 == planned.y0 &&
              st->bx1 == planned.x1() - 1 && st->by1 == planned.y1() - 1;
    if (!ok) st->box_mismatch = 1;
}

__global__ void k_snapshot_count(FoldStats* st, const CanvasCount* cc) {
    st->pv_count = cc->valid_count;
}

// |pano valid| before fold k from the claims' counts (hist[m]: pixels first
// covered by view m)
__global__ void k_count_from_hist(FoldStats* st, const unsigned long long* hist, int k) {
    unsigned long long c = 0;
    for (int m = 0; m < k; ++m) c += hist[m];
    st->pv_count = c;
}

// src/image.cpp:134-162 then src/image.cpp:70-83: crop of both sides over the
// Area3 box (invalid pixels zeroed) and their gray levels.
template <class V, class P>
__global__ void k_crop_gray(P pano, V view, Rect box, int ch, float* __restrict__ gl,
                            float* __restrict__ gr) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    int j = blockIdx.y;
    if (i >= box.w) return;
    int x = box.x0 + i, y = box.y0 + j;
    float4 l = pano.valid_at(x, y) ? pano.value_at(x, y) : make_float4(0.f, 0.f, 0.f, 0.f);
    float4 r = view.valid_at(x, y) ? view.value_at(x, y) : make_float4(0.f, 0.f, 0.f, 0.f);
    size_t o = (size_t)j * box.w + i;
    gl[o] = ch == 3 ? gray3(l.x, l.y, l.z) : l.x;
    gr[o] = ch == 3 ? gray3(r.x, r.y, r.z) : r.x;
}

// ============================================================================
// K1 — Gaussian pyramid (src/flow.cpp:29-56): one level of both images.
// out(i,j) = sum_t k[t] * tmp(2i, clamp(2j+t)),  tmp(x,y) = sum_s k[s] in(clamp(x+s), y)
// with float accumulation in tap order, exactly as the reference's two passes.
// ============================================================================
__global__ void k_downsample(const float* __restrict__ in0, const float* __restrict__ in1,
                             float* __restrict__ out0, float* __restrict__ out1, int w, int h,
                             int ow, int oh) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    int j = blockIdx.y * blockDim.y + threadIdx.y;
    if (i >= ow || j >= oh) return;
    const float* in = blockIdx.z == 0 ? in0 : in1;
    float* out = blockIdx.z == 0 ? out0 : out1;
    int xs[5];
#pragma unroll
    for (int s = -2; s <= 2; ++s) xs[s + 2] = clampi(2 * i + s, 0, w - 1);
    float acc = 0.f;
#pragma unroll
    for (int t = -2; t <= 2; ++t) {
        const float* row = in + (size_t)clampi(2 * j + t, 0, h - 1) * w;
        float tmp = 0.f;
#pragma unroll
        for (int s = 0; s < 5; ++s) tmp += binom_tap(s - 2) * __ldg(row + xs[s]);
        acc += binom_tap(t) * tmp;
    }
    out[(size_t)j * ow + i] = acc;
}

// K2+K3 (the fused LK iteration) lives in fs_lk.cu.

// ============================================================================
// K4 — flow smoothing (src/flow.cpp:113-130, 294-297): one or two fused 3x3
// truncated-mean passes of dx and dy; at level 0 also the final cap and the
// valid plane (src/flow.cpp:300-313).
// ============================================================================
constexpr int SM_TX = 32, SM_TY = 16;
__constant__ double kInvSmall[10] = {0.0,       1.0,       1.0 / 2, 1.0 / 3, 1.0 / 4,
                                     1.0 / 5,   1.0 / 6,   1.0 / 7, 1.0 / 8, 1.0 / 9};

// One 3x3 mean (src/flow.cpp:175-200): the in-image neighbours summed in
// double in the reference's row-major order, then (float)(sum / n).  INNER
// blocks lie (with their halo) inside the level, so every neighbour counts
// and n = 9.
template <bool INNER, int TW>
__device__ __forceinline__ float2 box3(const float2 (*tile)[TW], int ly, int lx, int gx, int gy,
                                       int w, int h) {
    double ax = 0.0, ay = 0.0;
    int n = 0;
#pragma unroll
    for (int dj = -1; dj <= 1; ++dj)
#pragma unroll
        for (int di = -1; di <= 1; ++di) {
            if (!INNER) {
                const int xx = gx + di, yy = gy + dj;
                if (xx < 0 || xx >= w || yy < 0 || yy >= h) continue;
            }
            const float2 v = tile[ly + dj][lx + di];
            ax += v.x;
            ay += v.y;
            ++n;
        }
    if (INNER) n = 9;
    return make_float2(div_to_float(ax, n, kInvSmall[n]), div_to_float(ay, n, kInvSmall[n]));
}

// Block of SM_TX x SM_TY threads, output tile SM_OX x SM_OY: the first pass
// covers the tile plus a 1-pixel ring — exactly one position per thread.
constexpr int SM_OX = SM_TX - 2, SM_OY = SM_TY - 2;

template <bool INNER>
__device__ __forceinline__ void smooth_tile(const SmoothArgs& a, float2 (*src)[SM_OX + 4],
                                            float2 (*p1)[SM_TX]) {
    const int d = blockIdx.z;
    const int w = a.w, h = a.h;
    const int bx = blockIdx.x * SM_OX, by = blockIdx.y * SM_OY;
    const int tx = threadIdx.x, ty = threadIdx.y;
    const bool two = a.passes == 2;
    if (two) {
        const int gx = bx - 1 + tx, gy = by - 1 + ty;
        float2 v = make_float2(0.f, 0.f);
        if (INNER || (gx >= 0 && gx < w && gy >= 0 && gy < h))
            v = box3<INNER, SM_OX + 4>(src, ty + 1, tx + 1, gx, gy, w, h);
        p1[ty][tx] = v;
        __syncthreads();
    }
    if (tx >= SM_OX || ty >= SM_OY) return;
    const int gx = bx + tx, gy = by + ty;
    if (gx >= w || gy >= h) return;
    const float2 v = two ? box3<INNER, SM_TX>(p1, ty + 1, tx + 1, gx, gy, w, h)
                         : box3<INNER, SM_OX + 4>(src, ty + 2, tx + 2, gx, gy, w, h);
    float vx = v.x, vy = v.y;
    const size_t o = (size_t)gy * w + gx;
    if (a.final_cap > 0.f) {
        final_cap(a.final_cap, vx, vy);
        (d ? a.valid_out[1] : a.valid_out[0])[o] = (d ? a.ok[1] : a.ok[0])[o];
    }
    (d ? a.fout[1] : a.fout[0])[o] = make_float2(vx, vy);
}

__global__ void __launch_bounds__(SM_TX* SM_TY, 3) k_smooth(SmoothArgs a) {
    __shared__ float2 src[SM_OY + 4][SM_OX + 4];
    __shared__ float2 p1[SM_TY][SM_TX];
    const int d = blockIdx.z;
    const float2* fin = d ? a.fin[1] : a.fin[0];
    const int w = a.w, h = a.h;
    const int bx = blockIdx.x * SM_OX, by = blockIdx.y * SM_OY;
    for (int t = threadIdx.y * SM_TX + threadIdx.x; t < (SM_OY + 4) * (SM_OX + 4);
         t += SM_TX * SM_TY) {
        const int ly = t / (SM_OX + 4), lx = t - ly * (SM_OX + 4);
        const int gx = bx - 2 + lx, gy = by - 2 + ly;
        float2 v = make_float2(0.f, 0.f);
        if (gx >= 0 && gx < w && gy >= 0 && gy < h) v = fin[(size_t)gy * w + gx];
        src[ly][lx] = v;
    }
    __syncthreads();
    if (bx >= 2 && by >= 2 && bx + SM_OX + 2 <= w && by + SM_OY + 2 <= h)
        smooth_tile<true>(a, src, p1);
    else
        smooth_tile<false>(a, src, p1);
}

// K4, column-sweep form: a CTA of S2_T threads owns S2_T - 4 output columns
// and S2_OY output rows.  The (S2_OY + 4) x S2_T input tile is staged once;
// each thread then walks one column down, carrying the two previous rows of
// its 3x3 window in registers as doubles (every staged float is widened once
// per window row instead of nine times), first for the pass-1 plane
// ((S2_OY + 2) x (S2_T - 2), staged in shared memory) and then for the
// output.  Out-of-image taps are staged as -0.0, the exact identity of
// double addition, so the reference's skip-and-count (src/flow.cpp:113-130)
// becomes a plain sum divided by (in-image rows) x (in-image columns).
constexpr int S2_T = 128;
#ifndef FS_SMOOTH_OY
#define FS_SMOOTH_OY 8
#endif
constexpr int S2_OY = FS_SMOOTH_OY;
#ifndef FS_SMOOTH2_MIN_PX
#define FS_SMOOTH2_MIN_PX 100000
#endif
constexpr int S2_OX = S2_T - 4;

// One column of 3x3 means: outputs q = 0..rows-1 read input rows q..q+2 at
// columns t..t+2.  gx/gy0: global position of output (0, this column).
template <bool INNER, class Sink>
__device__ __forceinline__ void sweep3(const float2 (*in)[S2_T], int t, int rows, int gx,
                                       int gy0, int w, int h, Sink sink) {
    double x0[3], y0[3], x1[3], y1[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const float2 a = in[0][t + k], b = in[1][t + k];
        x0[k] = a.x; y0[k] = a.y; x1[k] = b.x; y1[k] = b.y;
    }
    int ncol = 3;
    if (!INNER) ncol = 3 - (gx - 1 < 0) - (gx + 1 >= w);
#pragma unroll 4
    for (int q = 0; q < rows; ++q) {
        double x2[3], y2[3];
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            const float2 c = in[q + 2][t + k];
            x2[k] = c.x; y2[k] = c.y;
        }
        double ax = 0.0, ay = 0.0;
#pragma unroll
        for (int k = 0; k < 3; ++k) { ax += x0[k]; ay += y0[k]; }
#pragma unroll
        for (int k = 0; k < 3; ++k) { ax += x1[k]; ay += y1[k]; }
#pragma unroll
        for (int k = 0; k < 3; ++k) { ax += x2[k]; ay += y2[k]; }
        int n = 9;
        if (!INNER) {
            const int gy = gy0 + q;
            n = ncol * (3 - (gy - 1 < 0) - (gy + 1 >= h));
        }
        sink(q, div_to_float(ax, n, kInvSmall[n]), div_to_float(ay, n, kInvSmall[n]));
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            x0[k] = x1[k]; y0[k] = y1[k]; x1[k] = x2[k]; y1[k] = y2[k];
        }
    }
}

template <bool INNER>
__device__ __forceinline__ void smooth2_tile(const SmoothArgs& a, float2 (*src)[S2_T],
                                             float2 (*p1)[S2_T]) {
    const int d = blockIdx.z;
    const int w = a.w, h = a.h;
    const int bx = blockIdx.x * S2_OX, by = blockIdx.y * S2_OY;
    const int t = threadIdx.x;
    const float2 nz = make_float2(-0.f, -0.f);
    const float2(*last)[S2_T] = src;
    int lastoff = 0;  // the last pass reads columns t..t+2 of `last` at offset lastoff
    if (a.passes == 2) {
        if (t < S2_T - 2) {
            const int gx = bx - 1 + t;
            const bool colin = gx >= 0 && gx < w;
            sweep3<INNER>(src, t, S2_OY + 2, gx, by - 1, w, h, [&](int q, float vx, float vy) {
                const int gy = by - 1 + q;
                p1[q][t + 1] = (INNER || (colin && gy >= 0 && gy < h)) ? make_float2(vx, vy) : nz;
            });
        }
        __syncthreads();
        last = p1;
        lastoff = 1;
    }
    if (t >= S2_OX) return;
    const int gx = bx + t;
    if (gx >= w) return;
    float2* fo = d ? a.fout[1] : a.fout[0];
    const uint8_t* ok = d ? a.ok[1] : a.ok[0];
    uint8_t* vo = d ? a.valid_out[1] : a.valid_out[0];
    const int rows = min(S2_OY, h - by);
    sweep3<INNER>((const float2(*)[S2_T])(&last[0][lastoff]), t, rows, gx, by, w, h,
                  [&](int q, float vx, float vy) {
                      const size_t o = (size_t)(by + q) * w + gx;
                      if (a.final_cap > 0.f) {
                          final_cap(a.final_cap, vx, vy);
                          vo[o] = ok[o];
                      }
                      fo[o] = make_float2(vx, vy);
                  });
}

__global__ void __launch_bounds__(S2_T) k_smooth2(SmoothArgs a) {
    __shared__ float2 src[S2_OY + 4][S2_T];
    __shared__ float2 p1[S2_OY + 2][S2_T];
    const int d = blockIdx.z;
    const float2* fin = d ? a.fin[1] : a.fin[0];
    const int w = a.w, h = a.h;
    const int bx = blockIdx.x * S2_OX, by = blockIdx.y * S2_OY;
    const int t = threadIdx.x;
    // one pass reads the tile from row 1 (its outputs need rows by-1..)
    const int gx = bx - 2 + t;
    const bool colin = gx >= 0 && gx < w;
#pragma unroll
    for (int r = 0; r < S2_OY + 4; ++r) {
        const int gy = by - 2 + r;
        float2 v = make_float2(-0.f, -0.f);
        if (colin && gy >= 0 && gy < h) v = fin[(size_t)gy * w + gx];
        src[r][t] = v;
    }
    __syncthreads();
    const bool inner = bx >= 2 && by >= 2 && bx + S2_OX + 2 <= w && by + S2_OY + 2 <= h;
    if (a.passes == 2) {
        if (inner) smooth2_tile<true>(a, src, p1);
        else smooth2_tile<false>(a, src, p1);
    } else {
        // one pass: outputs read src rows q+1..q+3, columns t+1..t+3
        if (inner) smooth2_tile<true>(a, (float2(*)[S2_T])&src[1][1], p1);
        else smooth2_tile<false>(a, (float2(*)[S2_T])&src[1][1], p1);
    }
}

// Level-0 finalisation when smoothing_passes == 0 (src/flow.cpp:300-313).
__global__ void k_finalize_flow(SmoothArgs a) {
    const int d = blockIdx.z;
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    int n = a.w * a.h;
    if (i >= n) return;
    float2 f = (d ? a.fin[1] : a.fin[0])[i];
    final_cap(a.final_cap, f.x, f.y);
    (d ? a.fout[1] : a.fout[0])[i] = f;
    (d ? a.valid_out[1] : a.valid_out[0])[i] = (d ? a.ok[1] : a.ok[0])[i];
}

// ============================================================================
// K5/K6 — exact Euclidean distance transform (src/blend_field.cpp:19-86).
//
// Squared distances are integers, so any exact method reproduces the
// reference's sqrt(dt) bit for bit.  The transform is separable: pass 1 is a
// 1-D nearest-seed search along one axis (segmented so long lines run in
// parallel), pass 2 the lower envelope of parabolas along the other axis
// (Felzenszwalb, with exact int64 intersection comparisons, pruned at the
// nearest on-line seeds which dominate everything behind them).  Work is
// restricted to a domain W around the output box C; a per-pixel certificate
// proves that no seed outside W could be closer, otherwise the fold is
// flagged and recomputed on the full domain by the host.
// ============================================================================
constexpr int EDT_SEG = 64;
#ifndef EDT_BITS_RUN
#define EDT_BITS_RUN 4
#endif

template <class M>
__device__ __forceinline__ void edt_line_xy(const EdtJob<M>& J, int line, int p, int& x, int& y) {
    if (J.vfirst) {
        x = J.W.x0 + line;
        y = J.W.y0 + p;
    } else {
        x = J.W.x0 + p;
        y = J.W.y0 + line;
    }
}

// pass 1a: the seed mask of every (line, 64-position segment) as a bit set.
// Columns-first: a thread per (column, segment), consecutive threads read
// consecutive columns.  Rows-first: a warp per (row, segment), two ballots.
template <class M>
__global__ void k_edt_bits(EdtJob<M> J0, EdtJob<M> J1) {
    const EdtJob<M>& J = blockIdx.z == 0 ? J0 : J1;
    if (!J.active) return;
    const int nlines = J.vfirst ? J.W.w : J.W.h;
    const int len = J.vfirst ? J.W.h : J.W.w;
    const int nseg = (len + EDT_SEG - 1) / EDT_SEG;
    // rows-first: EDT_BITS_RUN consecutive segments of a row per warp (the job
    // selection and index set-up paid once per run); columns-first: one
    const int run = J.vfirst ? 1 : EDT_BITS_RUN;
    const int seg0 = blockIdx.y * run;
    const int seg1 = min(seg0 + run, nseg);
    if (J.vfirst) {
        const int line = blockIdx.x * blockDim.x + threadIdx.x;
        if (line >= nlines) return;
        for (int seg = seg0; seg < seg1; ++seg) {
            const int p0 = seg * EDT_SEG;
            const int n = min(EDT_SEG, len - p0);
            unsigned long long bits = 0;
#pragma unroll 16
            for (int k = 0; k < EDT_SEG; ++k) {
                if (k < n && J.mask(J.W.x0 + line, J.W.y0 + p0 + k)) bits |= 1ull << k;
            }
            J.bits[(size_t)seg * nlines + line] = bits;
        }
    } else {
        const int lane = threadIdx.x & 31;
        const int line = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
        if (line >= nlines) return;
        const int y = J.W.y0 + line;
        for (int seg = seg0; seg < seg1; ++seg) {
            const int pa = seg * EDT_SEG + lane, pb = pa + 32;
            const bool a = pa < len && J.mask(J.W.x0 + pa, y);
            const bool b = pb < len && J.mask(J.W.x0 + pb, y);
            const unsigned lo = __ballot_sync(0xffffffffu, a), hi = __ballot_sync(0xffffffffu, b);
            if (lane == 0)
                J.bits[(size_t)seg * nlines + line] =
                    (unsigned long long)lo | ((unsigned long long)hi << 32);
        }
    }
}

// pass 1b: squared 1-D distance to the nearest seed along the line, for every
// output position (C's extent along the line), from the segment bit sets.
template <class M>
__global__ void k_edt_line(EdtJob<M> J0, EdtJob<M> J1) {
    const EdtJob<M>& J = blockIdx.z == 0 ? J0 : J1;
    if (!J.active) return;
    const int nlines = J.vfirst ? J.W.w : J.W.h;
    const int len = J.vfirst ? J.W.h : J.W.w;
    const int nseg = (len + EDT_SEG - 1) / EDT_SEG;
    const int oa = J.vfirst ? J.C.y0 - J.W.y0 : J.C.x0 - J.W.x0;
    const int ob = oa + (J.vfirst ? J.C.h : J.C.w);
    const int line = blockIdx.x * blockDim.x + threadIdx.x;
    const int seg = oa / EDT_SEG + blockIdx.y;
    if (line >= nlines || seg >= nseg) return;
    const int s0 = seg * EDT_SEG;
    const int p0 = max(s0, oa), p1 = min(min(len, s0 + EDT_SEG), ob);
    if (p0 >= p1) return;
    const unsigned long long* B = J.bits + line;
    const unsigned long long mine = B[(size_t)seg * nlines];
    int prev = -(1 << 30), next = 1 << 30;  // nearest seed before / after the segment
    // nearest seeds outside the segment: four segments' masks per round trip
    for (int s = seg - 1; s >= 0; s -= 4) {
        unsigned long long m[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) m[j] = s - j >= 0 ? B[(size_t)(s - j) * nlines] : 0ull;
        int hit = -1;
#pragma unroll
        for (int j = 3; j >= 0; --j)
            if (m[j]) hit = j;
        if (hit >= 0) {
            prev = (s - hit) * EDT_SEG + 63 - __clzll((long long)m[hit]);
            break;
        }
    }
    for (int s = seg + 1; s < nseg; s += 4) {
        unsigned long long m[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) m[j] = s + j < nseg ? B[(size_t)(s + j) * nlines] : 0ull;
        int hit = -1;
#pragma unroll
        for (int j = 3; j >= 0; --j)
            if (m[j]) hit = j;
        if (hit >= 0) {
            next = (s + hit) * EDT_SEG + __ffsll((long long)m[hit]) - 1;
            break;
        }
    }
    const int gstride = J.vfirst ? J.W.w : J.W.h;  // pass-2 line length
    // walk the outputs with the nearest seeds at or before (last) and at or
    // after (nxt) p, advancing nxt past each seed it reaches
    const int k0 = p0 - s0;
    const unsigned long long below = k0 ? mine & ((1ull << k0) - 1) : 0ull;
    int last = below ? s0 + 63 - __clzll((long long)below) : prev;
    const unsigned long long from0 = mine & ~((1ull << k0) - 1);
    int nxt = from0 ? s0 + __ffsll((long long)from0) - 1 : next;
    int* gp = J.g + (size_t)(p0 - oa) * gstride + line;
    for (int p = p0; p < p1; ++p, gp += gstride) {
        if (p > nxt) {
            const unsigned long long hm = mine & ~((1ull << (p - s0)) - 1);
            nxt = hm ? s0 + __ffsll((long long)hm) - 1 : next;
        }
        if (nxt == p) last = p;
        const int d = min(p - last, nxt - p);
        *gp = d < 46341 ? d * d : kInfSq;
    }
}

// pass 2: lower envelope of parabolas along the other axis, a warp per output
// line: ballot search of the nearest on-line seeds around the output range
// (they dominate every site behind them), ballot compaction of the finite
// sites in between, envelope built by lane 0 with exact int64 intersection
// comparisons (Felzenszwalb, src/blend_field.cpp:19-47), then every lane
// evaluates its outputs by binary search over the envelope's breakpoints.
template <class M>
__global__ void k_edt_envelope(EdtJob<M> J0, EdtJob<M> J1, const FoldStats* st) {
    const EdtJob<M>& J = blockIdx.z == 0 ? J0 : J1;
    if (!J.active) return;
    const int nout_lines = J.vfirst ? J.C.h : J.C.w;
    const int L = J.vfirst ? J.W.w : J.W.h;  // sites per line
    const int lane = threadIdx.x & 31;
    const int ol = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (ol >= nout_lines) return;
    const int* f = J.g + (size_t)ol * L;
    int* stk = J.stack + (size_t)ol * L;
    const int qa = J.vfirst ? J.C.x0 - J.W.x0 : J.C.y0 - J.W.y0;
    const int qb = qa + (J.vfirst ? J.C.w : J.C.h);
    int lo = 0, hi = L - 1;
    for (int base = qa; base >= 0; base -= 32) {
        const int s = base - lane;
        const unsigned m = __ballot_sync(0xffffffffu, s >= 0 && f[s] == 0);
        if (m) {
            lo = base - (__ffs(m) - 1);
            break;
        }
    }
    for (int base = qb - 1; base < L; base += 32) {
        const int s = base + lane;
        const unsigned m = __ballot_sync(0xffffffffu, s < L && f[s] == 0);
        if (m) {
            hi = base + __ffs(m) - 1;
            break;
        }
    }
    int n = 0;
    const unsigned lt = (1u << lane) - 1;
    for (int base = lo; base <= hi; base += 32) {
        const int s = base + lane;
        const bool fin = s <= hi && f[s] < kInfSq;
        const unsigned m = __ballot_sync(0xffffffffu, fin);
        if (fin) stk[n + __popc(m & lt)] = s;
        n += __popc(m);
    }
    __syncwarp();
    int ne = 0;
    if (lane == 0) {
        // the top two stack entries (site t over u) and their g = f + s^2 in
        // registers, the next candidate's site and g loaded one step ahead:
        // a pop reads one entry back, a push writes one (the same exact int64
        // comparisons as the textbook loop)
        int t = 0, u = 0;
        long long gt = 0, gu = 0;
        int qn = n > 0 ? stk[0] : 0;
        long long fn = n > 0 ? f[qn] : 0;
        for (int i = 0; i < n; ++i) {
            const int q = qn;
            const long long gq = fn + (long long)q * q;
            if (i + 1 < n) {
                qn = stk[i + 1];
                fn = f[qn];
            }
            while (ne >= 2) {
                const long long n1 = gq - gt, d1 = 2LL * (q - t);
                const long long n2 = gt - gu, d2 = 2LL * (t - u);
                if (n1 * d2 > n2 * d1) break;
                --ne;  // t is hidden: u becomes the top
                t = u;
                gt = gu;
                if (ne >= 2) {
                    u = stk[ne - 2];
                    gu = (long long)f[u] + (long long)u * u;
                }
            }
            stk[ne++] = q;
            u = t;
            gu = gt;
            t = q;
            gt = gq;
        }
    }
    ne = __shfl_sync(0xffffffffu, ne, 0);
    __syncwarp();
    const bool have = J.which == 1   ? (st->pv_count - st->cnt3) > 0
                      : J.which == 2 ? st->cnt2 > 0
                                     : true;
    bool fail = false;
    for (int q = qa + lane; q < qb; q += 32) {
        int dsq = kInfSq;
        if (ne > 0) {
            // k = largest j with breakpoint z_j < q (z_0 = -inf)
            int klo = 0, khi = ne - 1;
            while (klo < khi) {
                const int mid = (klo + khi + 1) >> 1;
                const int a0 = stk[mid - 1], a1 = stk[mid];
                const long long num = ((long long)f[a1] + (long long)a1 * a1) -
                                      ((long long)f[a0] + (long long)a0 * a0);
                const long long den = 2LL * (a1 - a0);
                if (num < (long long)q * den)
                    klo = mid;
                else
                    khi = mid - 1;
            }
            const long long d = q - stk[klo];
            const long long v = d * d + f[stk[klo]];
            dsq = v < kInfSq ? (int)v : kInfSq;
        }
        int x, y;
        if (J.vfirst) {
            x = J.W.x0 + q;
            y = J.C.y0 + ol;
        } else {
            x = J.C.x0 + ol;
            y = J.W.y0 + q;
        }
        J.out[(size_t)(y - J.C.y0) * J.C.w + (x - J.C.x0)] = dsq;
        if (J.check && have) {  // distances to W's open edges are < 46341: squares fit in int
            int bnd = INT_MAX;
            if (!J.e_left) bnd = min(bnd, x - J.W.x0 + 1);
            if (!J.e_right) bnd = min(bnd, J.W.x1() - x);
            if (!J.e_top) bnd = min(bnd, y - J.W.y0 + 1);
            if (!J.e_bottom) bnd = min(bnd, J.W.y1() - y);
            if (bnd < 46341 && dsq > bnd * bnd) fail = true;  // (no open edge: INT_MAX)
        }
    }
    if (__any_sync(0xffffffffu, fail) && lane == 0)
        atomicOr((unsigned int*)&st->edt_fail, 1u << (blockIdx.z));
}

// ============================================================================
// K7 — Code 1 blend (src/blender.cpp:72-91) on the Area3 pixels of the crop
// box, and the composition onto the canvas (src/blender.cpp:66-71,
// src/pipeline.cpp:201-204).
// ============================================================================
template <int CH, class S>
__device__ __forceinline__ void bilinear_rgb(const S& s, int W, int H, double x, double y,
                                             float out[3]) {
    BiTap t = bi_tap(W, H, x, y);
    bool v[4];
    float4 px[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        v[k] = s.valid_at(t.xs[k], t.ys[k]);
        px[k] = v[k] ? s.value_at(t.xs[k], t.ys[k]) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    double wsum = 0.0;
#pragma unroll
    for (int k = 0; k < 4; ++k)
        if (v[k]) wsum += t.ws[k];
    if (wsum <= 0.0) {
        out[0] = out[1] = out[2] = 0.f;
        return;
    }
    double acc[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) {
        acc[c] = 0.0;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const float pv = c == 0 ? px[k].x : (c == 1 ? px[k].y : px[k].z);
            if (v[k]) acc[c] += t.ws[k] * pv;
        }
    }
    // all taps valid and the weights summing to exactly 1.0 (~97% of the
    // pixels): acc / 1.0 == acc, no division
    if (wsum == 1.0) {
#pragma unroll
        for (int c = 0; c < CH; ++c) out[c] = static_cast<float>(acc[c]);
    } else {
#pragma unroll
        for (int c = 0; c < CH; ++c) out[c] = static_cast<float>(acc[c] / wsum);
    }
}

// The panorama's validity before a fold: the canvas valid plane (serial
// folds), or the owner plane (owner < k: some earlier view covers the pixel)
// when the folds' Area2 copies are written ahead of the ordered chain.
struct PanoValidPlane {
    const uint8_t* valid;
    int w;
    __device__ __forceinline__ bool operator()(int x, int y) const {
        return valid[(size_t)y * w + x] != 0;
    }
};
struct PanoOwnerBefore {
    const uint8_t* owner;
    int w, k;
    __device__ __forceinline__ bool operator()(int x, int y) const {
        return owner[(size_t)y * w + x] < k;
    }
};
template <class PV>
struct CanvasSampler {
    const float4* rgb;
    PV pv;
    int w;
    __device__ __forceinline__ bool valid_at(int x, int y) const { return pv(x, y); }
    __device__ __forceinline__ float4 value_at(int x, int y) const { return rgb[(size_t)y * w + x]; }
};

#ifndef BLEND_MINB
#define BLEND_MINB 12  // 40 registers: 12 CTAs of 128 per SM (latency-bound gathers)
#endif
// LS: the sampler of L (the panorama before the fold) — the canvas, or
// (PanoHybrid) the first covering view's pixel where no earlier fold blended
// and the canvas only where one did, so first-cover pixels need no float copy
template <class V, class PV, int CH, class LS>
__global__ void __launch_bounds__(128, BLEND_MINB) k_blend_area3(Canvas cv, PV pv, V view, Rect box,
                                                     const float2* __restrict__ flr,
                              const float2* __restrict__ frl, const int* __restrict__ d1,
                              const int* __restrict__ d2, FoldStats* st, double k,
                              double coef, float4* __restrict__ out, float2* __restrict__ wgray,
                              const ReachCheck rc, const LS L, uchar4* __restrict__ canvas_out) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    int j = blockIdx.y;
    if (i >= box.w) return;
    int x = box.x0 + i, y = box.y0 + j;
    if (!(pv(x, y) && view.valid_at(x, y))) return;  // not Area3
    const bool have1 = (st->pv_count - st->cnt3) > 0, have2 = st->cnt2 > 0;
    size_t o = (size_t)j * box.w + i;
    double blend_r = eq1_area3(have1, have2, d1[o], d2[o]);
    double blend_l = 1.0 - blend_r;
    float2 rl = frl[o], lr = flr[o];
    float cl[3], cr[3];
    const double lx = x + rl.x * (1.0 - blend_l), ly = y + rl.y * (1.0 - blend_l);
    if (rc.on) {
        const BiTap t = bi_tap(cv.w, cv.h, lx, ly);
        bool bad = false;
#pragma unroll
        for (int q = 0; q < 4; ++q)
            if (pv(t.xs[q], t.ys[q]) && !rc.ok(t.xs[q], t.ys[q])) bad = true;
        if (bad) atomicOr(&st->reach_fail, 1u);
    }
    bilinear_rgb<CH>(L, cv.w, cv.h, lx, ly, cl);
    bilinear_rgb<CH>(view, cv.w, cv.h, x + lr.x * (1.0 - blend_r), y + lr.y * (1.0 - blend_r), cr);
    double mag_rl = sqrt((double)rl.x * rl.x + (double)rl.y * rl.y);
    double mag_lr = sqrt((double)lr.x * lr.x + (double)lr.y * lr.y);
    double sl, sr;
    softmax_weights(blend_l, blend_r, mag_rl, mag_lr, k, coef, sl, sr);
    float res[3] = {0.f, 0.f, 0.f};
#pragma unroll
    for (int c = 0; c < CH; ++c) {
        double v = cl[c] * sl + cr[c] * sr;
        res[c] = (float)clampd(v, 0.0, 1.0);
    }
    if (canvas_out)  // the fold's compose folded in: only the RGBA8 canvas (k_compose_area3)
        canvas_out[(size_t)y * cv.w + x] =
            quantize_px(make_float4(res[0], res[1], res[2], 0.f), cv.ch);
    else
        out[o] = make_float4(res[0], res[1], res[2], 0.f);
    if (wgray)  // gray of the warped constituents (warp_constituents, src/blender.cpp:150-158)
        wgray[o] = CH == 3 ? make_float2(gray3(cl[0], cl[1], cl[2]), gray3(cr[0], cr[1], cr[2]))
                           : make_float2(cl[0], cr[0]);
}

template <class V>
__global__ void k_compose(Canvas cv, V view, Rect box, const float4* __restrict__ blended,
                          CanvasCount* cc, const FoldStats* st) {
    int x = view.rect.x0 + blockIdx.x * blockDim.x + threadIdx.x;
    int y = view.rect.y0 + blockIdx.y;
    if (x >= view.rect.x1()) return;
    if (!view.valid_at(x, y)) return;
    size_t p = (size_t)y * cv.w + x;
    if (cv.valid[p]) {  // Area3
        cv.rgb[p] = blended[(size_t)(y - box.y0) * box.w + (x - box.x0)];
    } else {  // Area2
        cv.rgb[p] = view.value_at(x, y);
        cv.valid[p] = 1;
    }
}

// The compose split for the planned DAG: a fold's Area2 (the pixels its view
// covers first, owner == k: a copy of the view, src/blender.cpp:69-71) is
// written on the fold's branch as soon as the view is claimed; only its Area3
// (the blended box) is written in the ordered chain.
template <class V>
__global__ void __launch_bounds__(256) k_compose_area2(Canvas cv, V view,
                                                       const uint8_t* __restrict__ owner, int k,
                                                       uchar4* __restrict__ out, Rect r,
                                                       Rect cvr) {
    // 4 pixels per thread: one aligned word of the owner plane; rows strided
    // over the grid.  The 8-bit value of a view byte b is b itself
    // (lroundf((b * (1/255.f)) * 255.f) == b for every b: checked exhaustively).
    const float sc = 1.0f / 255.0f;
    for (int y = r.y0 + blockIdx.y; y < r.y1(); y += gridDim.y) {
        const size_t row = (size_t)y * cv.w;
        const int lead = (int)((row + (size_t)r.x0) & 3);
        const int x = r.x0 - lead + 4 * (int)(blockIdx.x * blockDim.x + threadIdx.x);
        if (x >= r.x1()) continue;
        const uchar4 o = *reinterpret_cast<const uchar4*>(owner + row + x);
        const bool m0 = o.x == k && x >= r.x0, m1 = o.y == k && x + 1 >= r.x0 && x + 1 < r.x1(),
                   m2 = o.z == k && x + 2 >= r.x0 && x + 2 < r.x1(), m3 = o.w == k && x + 3 < r.x1();
        if (!(m0 | m1 | m2 | m3)) continue;
        const uchar4* src = view.px + (size_t)(y - view.rect.y0) * view.rect.w + (x - view.rect.x0);
        const bool mine[4] = {m0, m1, m2, m3};
        uchar4 q[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) q[j] = mine[j] ? src[j] : make_uchar4(0, 0, 0, 0);
        const bool cv_row = y >= cvr.y0 && y < cvr.y1();
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            if (!mine[j]) continue;
            if (cv_row && x + j >= cvr.x0 && x + j < cvr.x1()) {  // the float canvas where it is read
                cv.rgb[row + x + j] = make_float4(q[j].x * sc, q[j].y * sc, q[j].z * sc, 0.f);
                cv.valid[row + x + j] = 1;
            }
            q[j].w = 255;
            if (cv.ch != 3) q[j].y = q[j].z = q[j].x;
        }
        if (!out) continue;
        if (m0 & m1 & m2 & m3) {  // the word is this view's: one store
            uint4 w4;
            w4.x = *reinterpret_cast<const unsigned int*>(&q[0]);
            w4.y = *reinterpret_cast<const unsigned int*>(&q[1]);
            w4.z = *reinterpret_cast<const unsigned int*>(&q[2]);
            w4.w = *reinterpret_cast<const unsigned int*>(&q[3]);
            *reinterpret_cast<uint4*>(out + row + x) = w4;
        } else {
#pragma unroll
            for (int j = 0; j < 4; ++j)
                if (mine[j]) out[row + x + j] = q[j];
        }
    }
}
template <class V>
__global__ void k_compose_area3(Canvas cv, V view, Rect box, const float4* __restrict__ blended,
                                const uint8_t* __restrict__ owner, int k,
                                uchar4* __restrict__ out, int write_cv) {
    const int x = box.x0 + blockIdx.x * blockDim.x + threadIdx.x;
    const int y = box.y0 + blockIdx.y;
    if (x >= box.x1()) return;
    const size_t p = (size_t)y * cv.w + x;
    if (owner[p] < k && view.valid_at(x, y)) {
        const float4 v = blended[(size_t)(y - box.y0) * box.w + (x - box.x0)];
        if (write_cv) cv.rgb[p] = v;
        if (out) out[p] = quantize_px(v, cv.ch);
    }
}

// validity-only fold step used by the planner: pano valid |= view valid
template <class V>
__global__ void k_union_valid(Canvas cv, V view) {
    int x = view.rect.x0 + blockIdx.x * blockDim.x + threadIdx.x;
    int y = view.rect.y0 + blockIdx.y;
    if (x >= view.rect.x1()) return;
    if (view.valid_at(x, y)) cv.valid[(size_t)y * cv.w + x] = 1;
}

// 4 owner bytes per thread (one aligned 32-bit word of the plane; bytes of
// the word outside the view are written back unchanged), rows strided over
// the grid; with `hist`, the claimed pixels are counted into hist[k] (one
// atomic per block).
__global__ void __launch_bounds__(256) k_claim_owner(uint8_t* __restrict__ owner, int w,
                                                     ViewU8 view, int k,
                                                     unsigned long long* __restrict__ hist) {
    __shared__ unsigned int red[8];
    unsigned int claimed = 0;
    for (int y = view.rect.y0 + blockIdx.y; y < view.rect.y1(); y += gridDim.y) {
        const size_t row = (size_t)y * w;
        const size_t f = ((row + view.rect.x0) & ~(size_t)3) +
                         4 * ((size_t)blockIdx.x * blockDim.x + threadIdx.x);
        if (f >= row + view.rect.x1()) continue;
        uchar4 o = *reinterpret_cast<const uchar4*>(owner + f);
        uint8_t b[4] = {o.x, o.y, o.z, o.w};
        const uchar4* src = view.px + (size_t)(y - view.rect.y0) * view.rect.w;
        unsigned int c = 0;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const long long x = (long long)(f + j) - (long long)row;
            if (x >= view.rect.x0 && x < view.rect.x1() && b[j] == 0xFF &&
                (view.all_valid || src[x - view.rect.x0].w >= 128)) {
                b[j] = (uint8_t)k;
                ++c;
            }
        }
        if (c) *reinterpret_cast<uchar4*>(owner + f) = make_uchar4(b[0], b[1], b[2], b[3]);
        claimed += c;
    }
    if (hist) {
        for (int d = 16; d; d >>= 1) claimed += __shfl_xor_sync(0xffffffffu, claimed, d);
        if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = claimed;
        __syncthreads();
        if (threadIdx.x == 0) {
            unsigned long long t = 0;
            for (int i = 0; i < 8; ++i) t += red[i];
            if (t) atomicAdd(&hist[k], t);
        }
    }
}

__global__ void k_count_update(CanvasCount* cc, const FoldStats* st) {
    cc->valid_count += st->cnt2;
}

// K8 — 8-bit RGBA output (src/image.cpp:52-65): alpha = valid.
__global__ void k_quantize(Canvas cv, Rect r, uchar4* __restrict__ out) {
    int x = r.x0 + blockIdx.x * blockDim.x + threadIdx.x;
    int y = r.y0 + blockIdx.y;
    if (x >= r.x1()) return;
    size_t p = (size_t)y * cv.w + x;
    uchar4 o = make_uchar4(0, 0, 0, 0);
    if (cv.valid[p]) {
        float4 v = cv.rgb[p];
        o.x = quantize8(v.x);
        o.y = cv.ch == 3 ? quantize8(v.y) : o.x;
        o.z = cv.ch == 3 ? quantize8(v.z) : o.x;
        o.w = 255;
    }
    out[p] = o;
}

// float output in ImageBuf layout (interleaved ch), invalid pixels are 0.
__global__ void k_export_float(Canvas cv, float* __restrict__ out, uint8_t* __restrict__ vout) {
    int x = blockIdx.x * blockDim.x + threadIdx.x;
    int y = blockIdx.y;
    if (x >= cv.w) return;
    size_t p = (size_t)y * cv.w + x;
    bool v = cv.valid[p] != 0;
    float4 px = v ? cv.rgb[p] : make_float4(0.f, 0.f, 0.f, 0.f);
    if (cv.ch == 3) {
        out[p * 3] = px.x;
        out[p * 3 + 1] = px.y;
        out[p * 3 + 2] = px.z;
    } else {
        out[p] = px.x;
    }
    vout[p] = v;
}

// ============================================================================
// Launch wrappers (host side)
// ============================================================================
namespace launch {

static inline dim3 row_grid(int w, int h, int bx = 256) { return dim3((w + bx - 1) / bx, h); }

template <class V>
void place_view(const Canvas& cv, const V& view, CanvasCount* count, cudaStream_t s, uchar4* out,
                bool write_cv) {
    k_place_view<<<row_grid(view.rect.w, (view.rect.h + PART_ROWS - 1) / PART_ROWS), 256, 0, s>>>(
        cv, view, count, out, write_cv ? 1 : 0);
}
template <class V, class P>
void partition(const P& pano, const V& view, FoldStats* st, cudaStream_t s) {
    k_partition<<<row_grid(view.rect.w, (view.rect.h + PART_ROWS - 1) / PART_ROWS), 256, 0, s>>>(
        pano, view, st);
}
void snapshot_count(FoldStats* st, const CanvasCount* cc, cudaStream_t s) {
    k_snapshot_count<<<1, 1, 0, s>>>(st, cc);
}
void check_box(FoldStats* st, const Rect& planned, cudaStream_t s) {
    k_check_box<<<1, 1, 0, s>>>(st, planned);
}
template <class V, class P>
void crop_gray(const P& pano, const V& view, const Rect& box, int ch, float* gl, float* gr,
               cudaStream_t s) {
    k_crop_gray<<<row_grid(box.w, box.h), 256, 0, s>>>(pano, view, box, ch, gl, gr);
}
void downsample(const float* in0, const float* in1, float* out0, float* out1, int w, int h,
                int nimg, cudaStream_t s) {
    int ow = max(1, w / 2), oh = max(1, h / 2);
    dim3 b(32, 8), g((ow + 31) / 32, (oh + 7) / 8, nimg);
    k_downsample<<<g, b, 0, s>>>(in0, in1, out0, out1, w, h, ow, oh);
}

void init() { lk_init(); }

void smooth(const SmoothArgs& a, cudaStream_t s) {
#ifdef FS_SMOOTH_TILE2D
    dim3 g((a.w + SM_OX - 1) / SM_OX, (a.h + SM_OY - 1) / SM_OY, a.ndir);
    k_smooth<<<g, dim3(SM_TX, SM_TY), 0, s>>>(a);
#else
    // small (coarse) levels keep the 2-D tiles: more CTAs for the few pixels
    if ((long long)a.w * a.h < FS_SMOOTH2_MIN_PX) {
        dim3 g((a.w + SM_OX - 1) / SM_OX, (a.h + SM_OY - 1) / SM_OY, a.ndir);
        k_smooth<<<g, dim3(SM_TX, SM_TY), 0, s>>>(a);
        return;
    }
    dim3 g((a.w + S2_OX - 1) / S2_OX, (a.h + S2_OY - 1) / S2_OY, a.ndir);
    k_smooth2<<<g, S2_T, 0, s>>>(a);
#endif
}
void finalize_flow(const SmoothArgs& a, cudaStream_t s) {
    int n = a.w * a.h;
    k_finalize_flow<<<dim3((n + 255) / 256, 1, a.ndir), 256, 0, s>>>(a);
}

template <class M>
void edt(const EdtJob<M>& j0, const EdtJob<M>& j1, const FoldStats* st, cudaStream_t s) {
    const EdtJob<M>* js[2] = {&j0, &j1};
    int max_lines = 0, max_seg = 0, max_oseg = 0, max_out = 0;
    for (auto* j : js) {
        if (!j->active) continue;
        int nlines = j->vfirst ? j->W.w : j->W.h;
        int len = j->vfirst ? j->W.h : j->W.w;
        int oa = j->vfirst ? j->C.y0 - j->W.y0 : j->C.x0 - j->W.x0;
        int olen = j->vfirst ? j->C.h : j->C.w;
        int nseg = (len + EDT_SEG - 1) / EDT_SEG;
        int oseg = (oa + olen - 1) / EDT_SEG - oa / EDT_SEG + 1;
        max_lines = max(max_lines, nlines);
        max_seg = max(max_seg, nseg);
        max_oseg = max(max_oseg, oseg);
        max_out = max(max_out, j->vfirst ? j->C.h : j->C.w);
    }
    if (max_lines == 0) return;
    // both jobs of a fold share the output box, hence the pass order
    const bool vf = j0.active ? j0.vfirst : j1.vfirst;
    if (vf)
        k_edt_bits<M><<<dim3((max_lines + 127) / 128, max_seg, 2), 128, 0, s>>>(j0, j1);
    else
        k_edt_bits<M><<<dim3((max_lines + 7) / 8, (max_seg + EDT_BITS_RUN - 1) / EDT_BITS_RUN, 2), 256, 0, s>>>(j0, j1);
    k_edt_line<M><<<dim3((max_lines + 127) / 128, max_oseg, 2), 128, 0, s>>>(j0, j1);
    k_edt_envelope<M><<<dim3((max_out + 7) / 8, 1, 2), 256, 0, s>>>(j0, j1, st);
}

template <class V>
void blend_area3(const Canvas& cv, const V& view, const Rect& box, const float2* flr,
                 const float2* frl, const int* d1, const int* d2, FoldStats* st, double k,
                 double coef, float4* out, float2* wgray, const uint8_t* owner, int fold,
                 cudaStream_t s, const ReachCheck* rc, const PanoViews* first_cover,
                 uchar4* canvas_out) {
    const ReachCheck r = rc ? *rc : ReachCheck{};
    const dim3 g = row_grid(box.w, box.h, 128);
#define FS_BLEND(PVT, LSV)                                                                    \
    do {                                                                                      \
        if (cv.ch == 3)                                                                       \
            k_blend_area3<V, PVT, 3><<<g, 128, 0, s>>>(cv, pv, view, box, flr, frl, d1, d2,   \
                                                      st, k, coef, out, wgray, r, LSV,       \
                                                      canvas_out);                            \
        else                                                                                  \
            k_blend_area3<V, PVT, 1><<<g, 128, 0, s>>>(cv, pv, view, box, flr, frl, d1, d2,   \
                                                      st, k, coef, out, wgray, r, LSV,       \
                                                      canvas_out);                            \
    } while (0)
    if (owner && first_cover) {
        const PanoOwnerBefore pv{owner, cv.w, fold};
        FS_BLEND(PanoOwnerBefore, (PanoHybrid{*first_cover, PanoPlane{cv.valid, cv.rgb, cv.w}}));
    } else if (owner) {
        const PanoOwnerBefore pv{owner, cv.w, fold};
        FS_BLEND(PanoOwnerBefore, (CanvasSampler<PanoOwnerBefore>{cv.rgb, pv, cv.w}));
    } else {
        const PanoValidPlane pv{cv.valid, cv.w};
        FS_BLEND(PanoValidPlane, (CanvasSampler<PanoValidPlane>{cv.rgb, pv, cv.w}));
    }
#undef FS_BLEND
}
template <class V>
void compose_area2(const Canvas& cv, const V& view, const uint8_t* owner, int fold,
                   cudaStream_t s, uchar4* out, const Rect* clip, const Rect* cv_clip) {
    Rect r = view.rect;
    if (clip) {  // the part of the view inside clip
        const int x0 = max(r.x0, clip->x0), y0 = max(r.y0, clip->y0);
        const int x1 = min(r.x1(), clip->x1()), y1 = min(r.y1(), clip->y1());
        r = Rect{x0, y0, x1 - x0, y1 - y0};
        if (r.w <= 0 || r.h <= 0) return;
    }
    const Rect cvr = cv_clip ? *cv_clip : Rect{0, 0, cv.w, cv.h};
    const int bx = ((r.w + 3) / 4 + 1 + 255) / 256;
    const int by = std::min(r.h, std::max(1, 148 * 8 / bx));
    k_compose_area2<<<dim3(bx, by), 256, 0, s>>>(cv, view, owner, fold, out, r, cvr);
}
void count_from_hist(FoldStats* st, const unsigned long long* hist, int k, cudaStream_t s) {
    k_count_from_hist<<<1, 1, 0, s>>>(st, hist, k);
}
template <class V>
void compose_area3(const Canvas& cv, const V& view, const Rect& box, const float4* blended,
                   const uint8_t* owner, int fold, cudaStream_t s, uchar4* out, bool write_cv) {
    k_compose_area3<<<row_grid(box.w, box.h), 256, 0, s>>>(cv, view, box, blended, owner, fold,
                                                          out, write_cv ? 1 : 0);
}
template <class V>
void compose(const Canvas& cv, const V& view, const Rect& box, const float4* blended,
             CanvasCount* cc, const FoldStats* st, cudaStream_t s) {
    k_compose<<<row_grid(view.rect.w, view.rect.h), 256, 0, s>>>(cv, view, box, blended, cc, st);
    k_count_update<<<1, 1, 0, s>>>(cc, st);
}
template <class V>
void union_valid(const Canvas& cv, const V& view, cudaStream_t s) {
    k_union_valid<<<row_grid(view.rect.w, view.rect.h), 256, 0, s>>>(cv, view);
}
// Host formats of the plan: RGB8 views (alpha implicitly 255) are expanded
// to RGBA8 on arrival; the RGBA8 canvas is packed to RGB8 before a read-back.
// 4 pixels per thread: 12 bytes in as three words, 16 out as one.
__global__ void __launch_bounds__(256) k_expand_rgb(const uint8_t* __restrict__ in,
                                                    uchar4* __restrict__ out, size_t n) {
    const size_t g = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    const size_t p0 = 4 * g;
    if (p0 >= n) return;
    if (p0 + 4 <= n) {
        const uint3 w = *reinterpret_cast<const uint3*>(in + 3 * p0);  // 12-byte aligned
        const uint8_t* b = reinterpret_cast<const uint8_t*>(&w);
        uint4 o;
        o.x = b[0] | (b[1] << 8) | (b[2] << 16) | 0xFF000000u;
        o.y = b[3] | (b[4] << 8) | (b[5] << 16) | 0xFF000000u;
        o.z = b[6] | (b[7] << 8) | (b[8] << 16) | 0xFF000000u;
        o.w = b[9] | (b[10] << 8) | (b[11] << 16) | 0xFF000000u;
        *reinterpret_cast<uint4*>(out + p0) = o;
    } else {
        for (size_t p = p0; p < n; ++p)
            out[p] = make_uchar4(in[3 * p], in[3 * p + 1], in[3 * p + 2], 255);
    }
}
// r: canvas rectangle; 4-pixel groups aligned in the flat canvas index, so
// the 12 output bytes of a group inside the rectangle are three words.
__global__ void __launch_bounds__(256) k_pack_rgb(const uchar4* __restrict__ in, int cw, Rect r,
                                                  uint8_t* __restrict__ out) {
    const int y = r.y0 + blockIdx.y;
    const size_t row = (size_t)y * cw;
    const size_t f = ((row + r.x0) & ~(size_t)3) + 4 * ((size_t)blockIdx.x * blockDim.x + threadIdx.x);
    if (f >= row + r.x1()) return;
    const long long x = (long long)f - (long long)row;
    if (x >= r.x0 && x + 4 <= r.x1()) {
        const uint4 q = *reinterpret_cast<const uint4*>(in + f);
        uint3 w;
        w.x = (q.x & 0xFFFFFFu) | (q.y << 24);
        w.y = ((q.y >> 8) & 0xFFFFu) | (q.z << 16);
        w.z = ((q.z >> 16) & 0xFFu) | (q.w << 8);
        *reinterpret_cast<uint3*>(out + 3 * f) = w;
    } else {
        for (int j = 0; j < 4; ++j) {
            if (x + j < r.x0 || x + j >= r.x1()) continue;
            const uchar4 q = in[f + j];
            out[3 * (f + j)] = q.x;
            out[3 * (f + j) + 1] = q.y;
            out[3 * (f + j) + 2] = q.z;
        }
    }
}
__global__ void __launch_bounds__(256) k_expand_rgb_rect(const uint8_t* __restrict__ in,
                                                         uchar4* __restrict__ out, int w, Rect r) {
    const int x = r.x0 + blockIdx.x * 64 + (threadIdx.x & 63);
    const int y = r.y0 + blockIdx.y * 4 + (threadIdx.x >> 6);
    if (x >= r.x1() || y >= r.y1()) return;
    const size_t i = (size_t)y * w + x;
    out[i] = make_uchar4(in[3 * i], in[3 * i + 1], in[3 * i + 2], 255);
}
__global__ void __launch_bounds__(256) k_set_alpha(uchar4* __restrict__ px, size_t n) {
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (size_t)gridDim.x * blockDim.x)
        px[i].w = 255;
}
void expand_rgb_rect(const uint8_t* in, uchar4* out, int w, const Rect& r, cudaStream_t s) {
    if (r.w > 0 && r.h > 0)
        k_expand_rgb_rect<<<dim3((r.w + 63) / 64, (r.h + 3) / 4), 256, 0, s>>>(in, out, w, r);
}
void set_alpha(uchar4* px, size_t n, cudaStream_t s) {
    if (n) k_set_alpha<<<(unsigned)std::min<size_t>((n + 255) / 256, 148 * 16), 256, 0, s>>>(px, n);
}
void expand_rgb(const uint8_t* in, uchar4* out, size_t n, cudaStream_t s) {
    if (n) k_expand_rgb<<<(unsigned)((n / 4 + 1 + 255) / 256), 256, 0, s>>>(in, out, n);
}
void pack_rgb(const uchar4* in, int cw, const Rect& r, uint8_t* out, cudaStream_t s) {
    if (r.w > 0 && r.h > 0)
        k_pack_rgb<<<dim3((unsigned)(((r.w + 3) / 4 + 1 + 255) / 256), r.h), 256, 0, s>>>(in, cw, r,
                                                                                          out);
}

__global__ void k_stamp(unsigned long long* t) {
    unsigned long long v;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(v));
    if (threadIdx.x == 0) *t = v;
}
void stamp(unsigned long long* slot, cudaStream_t s) { k_stamp<<<1, 32, 0, s>>>(slot); }
void claim_owner(uint8_t* owner, int w, const ViewU8& view, int k, cudaStream_t s,
                 unsigned long long* hist) {
    const int words = (view.rect.w + 3) / 4 + 1;  // the row's span may straddle one more word
    const int bx = (words + 255) / 256;
    const int by = std::min(view.rect.h, std::max(1, 148 * 8 / bx));
    k_claim_owner<<<dim3(bx, by), 256, 0, s>>>(owner, w, view, k, hist);
}
void quantize(const Canvas& cv, uchar4* out, cudaStream_t s) {
    quantize_rect(cv, Rect{0, 0, cv.w, cv.h}, out, s);
}
void quantize_rect(const Canvas& cv, const Rect& r, uchar4* out, cudaStream_t s) {
    if (r.w > 0 && r.h > 0) k_quantize<<<row_grid(r.w, r.h), 256, 0, s>>>(cv, r, out);
}
void export_float(const Canvas& cv, float* out, uint8_t* vout, cudaStream_t s) {
    k_export_float<<<row_grid(cv.w, cv.h), 256, 0, s>>>(cv, out, vout);
}

// explicit instantiations
template void union_valid<ViewU8>(const Canvas&, const ViewU8&, cudaStream_t);
template void place_view<ViewU8>(const Canvas&, const ViewU8&, CanvasCount*, cudaStream_t,
                                 uchar4*, bool);
template void place_view<ViewF4>(const Canvas&, const ViewF4&, CanvasCount*, cudaStream_t,
                                 uchar4*, bool);
template void partition<ViewU8, PanoPlane>(const PanoPlane&, const ViewU8&, FoldStats*,
                                           cudaStream_t);
template void partition<ViewU8, PanoViews>(const PanoViews&, const ViewU8&, FoldStats*,
                                           cudaStream_t);
template void partition<ViewF4, PanoPlane>(const PanoPlane&, const ViewF4&, FoldStats*,
                                           cudaStream_t);
template void crop_gray<ViewU8, PanoPlane>(const PanoPlane&, const ViewU8&, const Rect&, int,
                                           float*, float*, cudaStream_t);
template void crop_gray<ViewU8, PanoViews>(const PanoViews&, const ViewU8&, const Rect&, int,
                                           float*, float*, cudaStream_t);
template void crop_gray<ViewU8, PanoHybrid>(const PanoHybrid&, const ViewU8&, const Rect&, int,
                                           float*, float*, cudaStream_t);
template void crop_gray<ViewF4, PanoPlane>(const PanoPlane&, const ViewF4&, const Rect&, int,
                                           float*, float*, cudaStream_t);
template void edt<FoldMask<ViewU8, PanoViews>>(const EdtJob<FoldMask<ViewU8, PanoViews>>&,
                                               const EdtJob<FoldMask<ViewU8, PanoViews>>&,
                                               const FoldStats*, cudaStream_t);
template void edt<FoldMask<ViewU8, PanoPlane>>(const EdtJob<FoldMask<ViewU8, PanoPlane>>&,
                                               const EdtJob<FoldMask<ViewU8, PanoPlane>>&,
                                               const FoldStats*, cudaStream_t);
template void edt<FoldMask<ViewF4, PanoPlane>>(const EdtJob<FoldMask<ViewF4, PanoPlane>>&,
                                               const EdtJob<FoldMask<ViewF4, PanoPlane>>&,
                                               const FoldStats*, cudaStream_t);
template void edt<PlaneMask>(const EdtJob<PlaneMask>&, const EdtJob<PlaneMask>&,
                             const FoldStats*, cudaStream_t);
template void edt<LabelMask>(const EdtJob<LabelMask>&, const EdtJob<LabelMask>&,
                             const FoldStats*, cudaStream_t);
template void compose_area2<ViewU8>(const Canvas&, const ViewU8&, const uint8_t*, int,
                                    cudaStream_t, uchar4*, const Rect*, const Rect*);
template void compose_area3<ViewU8>(const Canvas&, const ViewU8&, const Rect&, const float4*,
                                    const uint8_t*, int, cudaStream_t, uchar4*, bool);
template void compose_area3<ViewF4>(const Canvas&, const ViewF4&, const Rect&, const float4*,
                                    const uint8_t*, int, cudaStream_t, uchar4*, bool);
template void blend_area3<ViewU8>(const Canvas&, const ViewU8&, const Rect&, const float2*,
                                  const float2*, const int*, const int*, FoldStats*, double,
                                  double, float4*, float2*, const uint8_t*, int, cudaStream_t,
                                  const ReachCheck*, const PanoViews*, uchar4*);
template void blend_area3<ViewF4>(const Canvas&, const ViewF4&, const Rect&, const float2*,
                                  const float2*, const int*, const int*, FoldStats*, double,
                                  double, float4*, float2*, const uint8_t*, int, cudaStream_t,
                                  const ReachCheck*, const PanoViews*, uchar4*);
template void compose<ViewU8>(const Canvas&, const ViewU8&, const Rect&, const float4*,
                              CanvasCount*, const FoldStats*, cudaStream_t);
template void compose<ViewF4>(const Canvas&, const ViewF4&, const Rect&, const float4*,
                              CanvasCount*, const FoldStats*, cudaStream_t);

}  // namespace launch
}  // namespace fs
