// K2+K3 — pyramidal LK iterations (src/flow.cpp:209-291), both directions.
//
// Per level the flow is refined by:
//   k_lk_prep   one thread per pixel: the level's starting flow (zero at the
//               coarsest level, else the fused 2x upsample of the coarser
//               flow, src/flow.cpp:138-170), its ever_ok, and the temporal
//               difference It = to(p + d) - from(p) (src/flow.cpp:248-249).
//   k_lk_sweep  one launch per iteration: window sums + 2x2 solve + update,
//               and, unless it is the level's last iteration, It for the next
//               iteration at the updated flow.
// Every gather of `to` thus happens in a per-pixel epilogue (independent
// loads, no dependent chain), and the sweep itself streams only coalesced
// loads.
//
// k_lk_sweep: a CTA owns an output tile of tw = 128 - 2r columns by th rows
// and sweeps its th + 2r input rows, warp-specialised:
//  producer warps 0-3 (thread c = input column x0 - r + c): per row the
//    central-difference gradient of `from` (src/flow.cpp:225-237) and It;
//    the exact double products enter the column's vertical running window
//    sums in registers.  (Ix, Iy, It) of the last 2r + 1 rows live in a
//    shared-memory ring so the row leaving the window is subtracted exactly.
//    Every NB rows the column sums are staged into one of two buffers.
//  consumer warps 4-7: horizontal (2r+1)-tap sums of a staged batch by
//    sliding runs of S outputs, the solve and update, the next It — while
//    the producers sweep the next batch.  Buffers are handed over with named
//    barriers (bar.arrive / bar.sync).
// FULL (a level's first iteration): five window sums, the eigenvalue test and
// the reference's division-form update (src/flow.cpp:267-291); it also stores
// the level-constant inverse structure tensor (c/det, b/det, a/det, ok) — the
// structure tensor depends only on the from-level gradients, so it and the
// eigenvalue decision are the same in every iteration of a level.  Later
// iterations form only the two mismatch sums and update by -(M^-1 b).
// Products are exact in double (float x float) and all window sums are double,
// agreeing with the reference's double prefix tables to ~1e-12 relative.
#include <algorithm>
#include <type_traits>

#include "fs_device.cuh"

namespace fs {

// Sweep modes: ITER (a later iteration: two mismatch sums, update by the
// stored inverse tensor), FULL (a level's first iteration in one pass: five
// sums, eigenvalue test, division-form update, stores the inverse tensor),
// TENSOR (the level-constant structure tensor alone: three sums, eigenvalue
// test, inverse tensor — no flow, so it runs off the coarse-to-fine chain),
// FIRST (an ITER that also writes the level's ever_ok from the TENSOR test).
enum { LK_ITER = 0, LK_FULL = 1, LK_TENSOR = 2, LK_FIRST = 3 };

#ifndef LK_MINB_FULL
#define LK_MINB_FULL 2
#endif
#ifndef LK_MINB_ITER
#define LK_MINB_ITER 3
#endif
#ifndef LK_MINB_F32
#define LK_MINB_F32 3
#endif
#ifndef LK_NS_F32
#define LK_NS_F32 2
#endif
#ifndef LK_IW_F32
#define LK_IW_F32 128
#endif

template <int M>
struct LkCfg {
    static constexpr bool FULL = M == LK_FULL;
    static constexpr int NQ = M == LK_FULL ? 5 : M == LK_TENSOR ? 3 : 2;  // window sums carried
#ifndef LK_NB_FULL
#define LK_NB_FULL 4
#define LK_S_FULL 4
#define LK_NB_ITER 4
#define LK_S_ITER 4
#endif
    static constexpr int NB = FULL ? LK_NB_FULL : LK_NB_ITER;  // rows per staged batch
    static constexpr int S = FULL ? LK_S_FULL : LK_S_ITER;     // outputs per horizontal run
    static constexpr bool GATHER = M != LK_TENSOR;              // It = T(p + d) - F(p)
    // Accumulation type.  FULL and TENSOR decide the level's valid bits (the
    // eigenvalue test) and keep the reference's double window sums; the
    // later iterations (ITER/FIRST) only refine a flow whose validity is
    // settled, and run in fp32: It by a float bilinear, products, window sums
    // and the update in float (well inside the 0.05 px mean-EPE budget;
    // -DFS_LK_ITER_F64 restores the double sweep).
#ifdef FS_LK_ITER_F64
    using Acc = double;
#else
    using Acc = std::conditional_t<M == LK_ITER || M == LK_FIRST, float, double>;
#endif
    static constexpr bool F32 = std::is_same<Acc, float>::value;
    // ring entries per column and row: FULL (Ix, Iy, It) and TENSOR (Ix, Iy)
    // as floats (products re-formed), ITER/FIRST the two products themselves
    static constexpr size_t RING = M == LK_FULL ? 3 * sizeof(float)
                                 : M == LK_TENSOR ? 2 * sizeof(float) : 2 * sizeof(Acc);
    static constexpr int MINB = F32 ? LK_MINB_F32 : M == LK_FULL ? LK_MINB_FULL : LK_MINB_ITER;
    // producer threads = input columns per CTA; 4 consumer warps.  The fp32
    // sweeps take 256 columns (240 outputs at r = 8: 7% halo columns, not
    // 14%) and run 2 CTAs/SM = 16 producer warps per SM.
    static constexpr int IW = F32 ? LK_IW_F32 : 128;
    static constexpr int THREADS = IW + 128;
    // staging buffers between producers and consumers (named barriers
    // 1..NS "staged", NS+1..2NS "released")
    static constexpr int NS = F32 ? LK_NS_F32 : 2;
};

#ifndef LK_CARRY_FULL
#define LK_CARRY_FULL 1
#endif

// Staged sums: plane [q][batch row][column].  Double modes: an odd row
// stride, so the consumers (consecutive threads = consecutive batch rows,
// then runs) read without bank conflicts and with plain column offsets.
// fp32 modes: one consumer warp per batch row reads its row as float4s (row
// stride 128, 16-byte aligned).
template <int M>
__host__ __device__ constexpr int lk_iwp() { return LkCfg<M>::F32 ? LkCfg<M>::IW : LkCfg<M>::IW + 1; }
// Ring of the last 2r+1 rows per column, so the row leaving the window is
// subtracted exactly: FULL keeps (Ix, Iy, It) as floats (five products are
// re-formed), later iterations keep the two double products themselves.
template <int M>
__host__ __device__ inline size_t lk_ring_bytes(int r) {
    return ((size_t)(2 * r + 1) * LkCfg<M>::IW * LkCfg<M>::RING + 15) & ~size_t(15);
}
template <int M>
__host__ __device__ inline size_t lk_stage_elems() {
    return (size_t)LkCfg<M>::NB * LkCfg<M>::NQ * lk_iwp<M>();
}
// fp32 sweeps: the four bilinear taps of every window pixel are copied
// (cp.async) into shared memory one batch ahead: [buffer][row][tap][column]
template <int M>
__host__ __device__ inline size_t lk_tap_bytes() {
    return LkCfg<M>::F32 ? (size_t)2 * LkCfg<M>::NB * 4 * LkCfg<M>::IW * sizeof(float) : 0;
}
// FS_CHECKS: the producer / consumer hand-off stamps (batch index last
// staged / released per buffer) and, for the fp32 sweeps, each tap slot's
// source offset, behind everything else
constexpr size_t kLkCheckBytes =
#ifdef FS_CHECKS
    256 + 2 * 4 * LK_IW_F32 * 3 * sizeof(int);
#else
    0;
#endif
template <int M>
__host__ __device__ inline size_t lk_check_off(int r);
template <int M>
__host__ inline size_t lk_smem_bytes(int r) {
    return kLkCheckBytes + lk_ring_bytes<M>(r) +
           LkCfg<M>::NS * lk_stage_elems<M>() * sizeof(typename LkCfg<M>::Acc) +
           lk_tap_bytes<M>();
}

template <int NT>
__device__ __forceinline__ void bar_sync(int id) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "n"(NT) : "memory");
}
template <int NT>
__device__ __forceinline__ void bar_arrive(int id) {
    asm volatile("bar.arrive %0, %1;" ::"r"(id), "n"(NT) : "memory");
}

// sample_level's clamp and taps (src/flow.cpp:100-111) at the float position
// (i + dx, j + dy) of src/flow.cpp:248: the clamp bounds are integers, so
// clamping, flooring and x - floor(x) are exact in float — the same taps and
// fractions as the reference's double evaluation.
struct TapF {
    int off, dx, dy;  // T offset of (x0, y0); +x / +y tap steps
    float fx, fy;
    int x0, y0;
};
__device__ __forceinline__ TapF level_tap_f(int w, int h, float px, float py) {
    const float wm = (float)(w - 1), hm = (float)(h - 1);
    px = px < 0.f ? 0.f : (wm < px ? wm : px);
    py = py < 0.f ? 0.f : (hm < py ? hm : py);
    const int x0 = (int)px, y0 = (int)py;
    TapF t;
    t.off = y0 * w + x0;
    t.dx = min(x0 + 1, w - 1) - x0;
    t.dy = (min(y0 + 1, h - 1) - y0) * w;
    t.fx = px - (float)x0;
    t.fy = py - (float)y0;
    t.x0 = x0;
    t.y0 = y0;
    return t;
}

// ---- per-level start: flow and ever_ok --------------------------------------
// A thread owns one column and LK_PREP_ROWS rows 8 apart: the column half of
// the align-centres tap (src/flow.cpp:150-157: x0, x1, fx, nearest xn) is
// computed once, the row half per row (uniform across the warp), and the four
// bilinear weights once per pixel for both components — the same expressions
// in the same order as src/flow.cpp:158-166, so the values are unchanged.
#ifndef LK_PREP_ROWS
#define LK_PREP_ROWS 4
#endif
template <int MODE>  // 0: zero flow (coarsest level), 2: upsample the coarser level
__global__ void __launch_bounds__(256) k_lk_prep(LkArgs a) {
    const LkDir& D = a.d[blockIdx.z];
    const int x = blockIdx.x * 32 + (threadIdx.x & 31);
    if (x >= a.w) return;
    const int yb = blockIdx.y * (8 * LK_PREP_ROWS) + (threadIdx.x >> 5);
    int x0 = 0, x1 = 0, xn = 0;
    double fx = 0.0;
    if (MODE == 2) {
        const double xc = clampd((x + 0.5) * a.sx - 0.5, 0.0, a.cw - 1.0);
        x0 = static_cast<int>(xc);
        x1 = imin(x0 + 1, a.cw - 1);
        fx = xc - x0;
        xn = clampi(static_cast<int>(lround(xc)), 0, a.cw - 1);
    }
#pragma unroll
    for (int k = 0; k < LK_PREP_ROWS; ++k) {
        const int y = yb + 8 * k;
        if (y >= a.h) return;
        float2 f = make_float2(0.f, 0.f);
        uint8_t ok = 0;
        if (MODE == 2) {
            const double yc = clampd((y + 0.5) * a.sy - 0.5, 0.0, a.ch - 1.0);
            const int y0 = static_cast<int>(yc);
            const int y1 = imin(y0 + 1, a.ch - 1);
            const double fy = yc - y0;
            const int yn = clampi(static_cast<int>(lround(yc)), 0, a.ch - 1);
            const float2* r0 = D.fin + (size_t)y0 * a.cw;
            const float2* r1 = D.fin + (size_t)y1 * a.cw;
            const float2 f00 = __ldg(r0 + x0), f10 = __ldg(r0 + x1);
            const float2 f01 = __ldg(r1 + x0), f11 = __ldg(r1 + x1);
            const double w00 = (1 - fx) * (1 - fy), w10 = fx * (1 - fy);
            const double w01 = (1 - fx) * fy, w11 = fx * fy;
            const double lx = w00 * f00.x + w10 * f10.x + w01 * f01.x + w11 * f11.x;
            const double ly = w00 * f00.y + w10 * f10.y + w01 * f01.y + w11 * f11.y;
            f = make_float2(static_cast<float>(2.0 * lx), static_cast<float>(2.0 * ly));
            ok = __ldg(D.okin + (size_t)yn * a.cw + xn);
        }
        const size_t o = (size_t)y * a.w + x;
        D.fout[o] = f;
        D.okout[o] = ok;
    }
}

// (v + a * b) for operands widened from float: the product is exact in double
// (24 + 24 bits), so the fused form rounds once, like the separate multiply
// and add it replaces (bit-identical, one instruction fewer).
__device__ __forceinline__ double lk_fma(double a, double b, double v) {
#ifdef FS_LK_NO_FMA
    return v + a * b;
#else
    return __fma_rn(a, b, v);
#endif
}

// ---- producer: sweep rows, stage vertical window sums ----------------------
// Per column, `from` walks down in registers: rows y-1, y (fu, f0) carried
// from the previous batch, rows y+1.. loaded one batch ahead (fn).  The
// horizontal neighbours F(x -/+ 1, y) are the neighbouring threads' centre
// values (their columns are clamp(x -/+ 1), src/flow.cpp:230-235); only the
// warp's edge lanes load them.  It = to(p + d) - from(p) (src/flow.cpp:248-249)
// is gathered at every window pixel from the current flow (loaded one batch
// ahead).  All indices are 32-bit (levels hold < 2^31 pixels).
template <int M>
__device__ __forceinline__ void lk_produce(const LkArgs& a, const LkDir& D, void* ringv,
                                           typename LkCfg<M>::Acc* stage, int x0, int ystart,
                                           int yend, int nbat) {
    using Cfg = LkCfg<M>;
    using Acc = typename Cfg::Acc;
    using Acc2 = std::conditional_t<Cfg::F32, float2, double2>;
    constexpr int NB = Cfg::NB, NQ = Cfg::NQ;
    constexpr bool FULL = Cfg::FULL, GATHER = Cfg::GATHER, TENSOR = M == LK_TENSOR;
    const int r = a.r, K = 2 * r + 1, w = a.w, h = a.h;
    constexpr int IWP = lk_iwp<M>(), IW = Cfg::IW, NT = Cfg::THREADS;
    const int c = threadIdx.x, lane = c & 31;
    const int x = x0 - r + c;
    const bool xin = x >= 0 && x < w;
    const int xc = clampi(x, 0, w - 1);
    const int dxl = clampi(x - 1, 0, w - 1) - xc, dxr = clampi(x + 1, 0, w - 1) - xc;
    const float* __restrict__ Fc = D.F + xc;
    const float2* __restrict__ Uc = D.fin + xc;
    const float* __restrict__ T = D.T;
    float* ringf = static_cast<float*>(ringv);
    Acc2* ringd = static_cast<Acc2*>(ringv);
    for (int k = 0; k < K; ++k) {
        if (FULL) {
            float* rs = ringf + (k * IW + c) * 3;
            rs[0] = rs[1] = rs[2] = 0.f;
        } else if (TENSOR) {
            float* rs = ringf + (k * IW + c) * 2;
            rs[0] = rs[1] = 0.f;
        } else {
            ringd[k * IW + c] = Acc2{0, 0};
        }
    }
    Acc V[NQ];
#pragma unroll
    for (int q = 0; q < NQ; ++q) V[q] = 0.0;
#ifdef FS_CHECKS
    extern __shared__ __align__(16) unsigned char smem[];
    int* chk = reinterpret_cast<int*>(smem + lk_check_off<M>(a.r));
    if (c == 0)
        for (int k = 0; k < 16; ++k) chk[k] = -1;
#endif
    auto ro = [&](int y) { return clampi(y, 0, h - 1) * w; };
    float2 fl[NB];
    if (GATHER) {
#pragma unroll
        for (int b = 0; b < NB; ++b) fl[b] = Uc[ro(ystart + b)];
    }
    // The column of `from` walks down in registers: cen[j] = F(x, clamp(y))
    // for y = ybase - 1 .. ybase + NB (the vertical gradient's rows), the
    // next batch's rows loaded one batch ahead.  (The double later-iteration
    // build, at 80 registers, reloads them instead.)
    constexpr bool CARRY = FULL ? LK_CARRY_FULL != 0 : (Cfg::F32 || TENSOR);
    float cen[CARRY ? NB + 2 : 1];
    if (CARRY) {
#pragma unroll
        for (int j = 0; j < NB + 2; ++j) cen[j] = __ldg(Fc + ro(ystart - 1 + j));
    }
    int slot = 0;
    for (int i = 0; i < nbat; ++i) {
        const int buf = i & 1;
        const int ybase = ystart + i * NB;
        float gxs[NB], gys[NB], dts[NB], tap[NB][4], tfx[NB], tfy[NB], ctr[NB], edge[NB];
        bool in[NB];
        // batches whose rows (and rows -1, +1) lie inside the level and the
        // band need no row clamps or row tests
        auto loads = [&](auto inner_t) {
            constexpr bool INNER = decltype(inner_t)::value;
            const float* Fb = Fc + (INNER ? ybase * w : 0);
#pragma unroll
            for (int b = 0; b < NB; ++b) {  // independent loads of the batch
                const int y = ybase + b;
                in[b] = INNER ? xin : (xin && y >= 0 && y < h && y < yend);
                const int yy = INNER ? y : clampi(y, 0, h - 1);
                const float* Fr = INNER ? Fb + b * w : Fc + yy * w;
                // F(clamp(x -/+ 1), y) are the adjacent lanes' centres (their
                // columns are x -/+ 1, clamped alike); the warp's edge lanes
                // load theirs (the horizontal gradient is formed below)
                edge[b] = 0.f;
                if (lane == 0 || lane == 31) edge[b] = __ldg(Fr + (lane == 0 ? dxl : dxr));
                if (CARRY) {
                    gys[b] = 0.5f * (cen[b + 2] - cen[b]);
                    ctr[b] = cen[b + 1];
                } else {
                    gys[b] = INNER ? 0.5f * (__ldg(Fr + w) - __ldg(Fr - w))
                                   : 0.5f * (__ldg(Fc + ro(y + 1)) - __ldg(Fc + ro(y - 1)));
                    ctr[b] = __ldg(Fr);
                }
                if (GATHER) {
                    const TapF t = level_tap_f(w, h, (float)xc + fl[b].x, (float)yy + fl[b].y);
                    tfx[b] = t.fx;
                    tfy[b] = t.fy;
                    const float* p = T + t.off;
                    tap[b][0] = __ldg(p);
                    tap[b][1] = __ldg(p + t.dx);
                    tap[b][2] = __ldg(p + t.dy);
                    tap[b][3] = __ldg(p + (t.dy + t.dx));
                }
            }
        };
        if (ybase >= 1 && ybase + NB <= h - 1 && ybase + NB <= yend)
            loads(std::true_type{});
        else
            loads(std::false_type{});
        if (i + 1 < nbat) {
            if (GATHER) {
#pragma unroll
                for (int b = 0; b < NB; ++b) fl[b] = Uc[ro(ybase + NB + b)];
            }
            if (CARRY) {
                cen[0] = cen[NB];
                cen[1] = cen[NB + 1];
#pragma unroll
                for (int j = 2; j < NB + 2; ++j) cen[j] = __ldg(Fc + ro(ybase + NB - 1 + j));
            }
        }
#pragma unroll
        for (int b = 0; b < NB; ++b) {  // src/flow.cpp:230-235, 0.5f * (F[i+1] - F[i-1])
            float lf = __shfl_up_sync(0xffffffffu, ctr[b], 1);
            float rt = __shfl_down_sync(0xffffffffu, ctr[b], 1);
            if (lane == 0) lf = edge[b];
            if (lane == 31) rt = edge[b];
            gxs[b] = 0.5f * (rt - lf);
        }
        if (GATHER) {
#pragma unroll
            for (int b = 0; b < NB; ++b) {
                if (Cfg::F32) {  // float bilinear (lerp form) of the same taps
                    const float u = __fmaf_rn(tfx[b], tap[b][1] - tap[b][0], tap[b][0]);
                    const float v = __fmaf_rn(tfx[b], tap[b][3] - tap[b][2], tap[b][2]);
                    dts[b] = __fmaf_rn(tfy[b], v - u, u) - ctr[b];
                } else {
                    LevelTap t;
                    t.fx = tfx[b];
                    t.fy = tfy[b];
                    dts[b] = level_combine(t, tap[b][0], tap[b][1], tap[b][2], tap[b][3]) - ctr[b];
                }
            }
        }
        if (i >= 2) bar_sync<NT>(3 + buf);  // consumers released this buffer
#ifdef FS_CHECKS
        if (i >= 2) FS_DCHECK(chk[8 + buf] == i - 2);
#endif
        Acc* st = stage + (size_t)buf * lk_stage_elems<M>();
#pragma unroll
        for (int b = 0; b < NB; ++b) {
            const double ix = in[b] ? gxs[b] : 0.f, iy = in[b] ? gys[b] : 0.f;
            const double tt = (GATHER && in[b]) ? dts[b] : 0.f;
            if (TENSOR) {
                float* rs = ringf + (slot * IW + c) * 2;
                const double ogx = rs[0], ogy = rs[1];
                rs[0] = (float)ix;
                rs[1] = (float)iy;
                V[0] = lk_fma(-ogx, ogx, lk_fma(ix, ix, V[0]));
                V[1] = lk_fma(-ogx, ogy, lk_fma(ix, iy, V[1]));
                V[2] = lk_fma(-ogy, ogy, lk_fma(iy, iy, V[2]));
            } else if (FULL) {
                float* rs = ringf + (slot * IW + c) * 3;
                const double ogx = rs[0], ogy = rs[1], odt = rs[2];
                rs[0] = (float)ix;
                rs[1] = (float)iy;
                rs[2] = (float)tt;
                V[0] = lk_fma(-ogx, ogx, lk_fma(ix, ix, V[0]));
                V[1] = lk_fma(-ogx, ogy, lk_fma(ix, iy, V[1]));
                V[2] = lk_fma(-ogy, ogy, lk_fma(iy, iy, V[2]));
                V[3] = lk_fma(-ogx, odt, lk_fma(ix, tt, V[3]));
                V[4] = lk_fma(-ogy, odt, lk_fma(iy, tt, V[4]));
            } else {
                Acc2* rp = ringd + (slot * IW + c);
                const Acc2 o = *rp;
                const float fxx = in[b] ? gxs[b] : 0.f, fyy = in[b] ? gys[b] : 0.f;
                const float ftt = in[b] ? dts[b] : 0.f;
                const Acc px = (Acc)fxx * (Acc)ftt, py = (Acc)fyy * (Acc)ftt;  // double: exact
                *rp = Acc2{px, py};
                V[0] = (V[0] + px) - o.x;
                V[1] = (V[1] + py) - o.y;
            }
            slot = slot + 1 == K ? 0 : slot + 1;
            Acc* vb = st + b * IWP + c;
#pragma unroll
            for (int q = 0; q < NQ; ++q) vb[q * NB * IWP] = V[q];
        }
#ifdef FS_CHECKS
        if (c == 0) chk[buf] = i;
#endif
        bar_arrive<NT>(1 + buf);  // batch staged
    }
}

#ifdef FS_CHECKS
// fault injection for the checks build's own test (fs_debug_inject): 1 = the
// producers mis-stamp every staged batch, 2 = they skip the cp.async wait
static __device__ int g_fs_inject;
#endif

// ---- producer (fp32 later iterations): a software pipeline ---------------
// Batch i's taps were issued (cp.async into shared memory) during batch i-1,
// from the flow loaded during batch i-2; its `from` rows (cen) and the warp
// edge lanes' horizontal neighbours were loaded during batch i-1.  So a batch
// starts with its data on chip: gradients, It (float bilinear of the staged
// taps), the two products, the column's running window sums (the row leaving
// the window comes from the ring of the last 2r + 1 products), staging.
// Batches whose preloaded rows all lie inside the level address them from one
// row offset (no per-row clamps); only the first and last batches of a
// column clamp.  CERT (row/column tiles only) adds the tap certificate.
__device__ __forceinline__ void cp_async4(uint32_t dst, const float* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

template <int M, bool CERT>
__device__ __forceinline__ void lk_produce_f32(const LkArgs& a, const LkDir& D, float2* ring,
                                               float* stage, float* tapb, int x0, int ystart,
                                               int yend, int nbat) {
    using Cfg = LkCfg<M>;
    constexpr int NB = Cfg::NB, IW = Cfg::IW, NT = Cfg::THREADS, IWP = lk_iwp<M>(), NS = Cfg::NS;
    const int r = a.r, K = 2 * r + 1, w = a.w, h = a.h;
    const int c = threadIdx.x, lane = c & 31;
    const int x = x0 - r + c;
    const bool xin = x >= 0 && x < w;
    const int xc = clampi(x, 0, w - 1);
    const float xcf = (float)xc, wm = (float)(w - 1), hm = (float)(h - 1);
    // warp edge lanes: the horizontal neighbour outside the warp (others: own column)
    const int eoff = lane == 0 ? clampi(x - 1, 0, w - 1) - xc
                   : lane == 31 ? clampi(x + 1, 0, w - 1) - xc : 0;
    const float* __restrict__ Fc = D.F + xc;
    const float2* __restrict__ Uc = D.fin + xc;
    const float* __restrict__ T = D.T;
    for (int k = 0; k < K; ++k) ring[k * IW + c] = make_float2(0.f, 0.f);
    float2* rp = ring + c;  // this column's ring slot the next input row replaces
    float2* const rend = ring + c + K * IW;
    const unsigned yhi = (unsigned)min(h, yend);  // rows with products: [0, yhi)
    float V0 = 0.f, V1 = 0.f;
    auto ro = [&](int y) { return clampi(y, 0, h - 1) * w; };
#ifdef FS_CHECKS
    extern __shared__ __align__(16) unsigned char smem[];
    int* chk = reinterpret_cast<int*>(smem + lk_check_off<M>(a.r));  // staged[8], freed[8]
    int* chk_tap = chk + 64;  // [buffer][row][column][off, dx, dy]
    if (c == 0)
        for (int k = 0; k < 16; ++k) chk[k] = -1;
#endif
    const uint32_t tap0 = (uint32_t)__cvta_generic_to_shared(tapb + c);
    // issue the taps of the batch starting at row yb into tap buffer tbuf
    // (src/flow.cpp:100-111 at (i + dx, j + dy), :248): the clamp bounds are
    // integers, so clamp / truncate / fraction are exact in float
    auto stage_taps = [&](int yb, int tbuf, const float2* fl, float* fx, float* fy) {
        const uint32_t d0 = tap0 + (uint32_t)(tbuf * NB * 4 * IW * 4);
#pragma unroll
        for (int b = 0; b < NB; ++b) {
            const int yy = clampi(yb + b, 0, h - 1);
            const float rx = xcf + fl[b].x, ry = (float)yy + fl[b].y;
            const float px = fminf(fmaxf(rx, 0.f), wm), py = fminf(fmaxf(ry, 0.f), hm);
            const int ix = (int)px, iy = (int)py;
            fx[b] = px - (float)ix;
            fy[b] = py - (float)iy;
            if (CERT) {  // a tile: this pixel's taps inside the exact pyramid part?
                // (the position before the clamp: at a cut the clamp itself
                // would differ from the untiled sample)
                const int q = a.cert_axis ? yb + b : x;
                const float raw = a.cert_axis ? ry : rx;
                if (xin && yb + b >= 0 && yb + b < h && q >= a.zlo && q < a.zhi &&
                    !(raw >= (float)a.exlo && raw <= (float)(a.exhi - 1)))
                    atomicOr(a.cert_fail, 1u);
            }
            const int dx = ix < w - 1 ? 1 : 0, dyw = iy < h - 1 ? w : 0;
            const float* p = T + (iy * w + ix);
            const uint32_t d = d0 + (uint32_t)(b * 4 * IW * 4);
#ifdef FS_CHECKS
            FS_DCHECK(iy * w + ix >= 0 && iy * w + ix + dyw + dx < w * h);
            int* ct = chk_tap + (((tbuf * NB + b) * IW) + c) * 3;
            ct[0] = iy * w + ix;
            ct[1] = dx;
            ct[2] = dyw;
#endif
            cp_async4(d, p);
            cp_async4(d + IW * 4, p + dx);
            cp_async4(d + 2 * IW * 4, p + dyw);
            cp_async4(d + 3 * IW * 4, p + (dyw + dx));
        }
        cp_async_commit();
    };
    float2 fl[NB];
    float tfx[NB], tfy[NB], cen[NB + 2], edg[NB];
#pragma unroll
    for (int b = 0; b < NB; ++b) fl[b] = Uc[ro(ystart + b)];
    stage_taps(ystart, 0, fl, tfx, tfy);
    if (nbat > 1) {
#pragma unroll
        for (int b = 0; b < NB; ++b) fl[b] = Uc[ro(ystart + NB + b)];
    }
#pragma unroll
    for (int j = 0; j < NB + 2; ++j) cen[j] = __ldg(Fc + ro(ystart - 1 + j));
#pragma unroll
    for (int b = 0; b < NB; ++b) edg[b] = __ldg(Fc + ro(ystart + b) + eoff);
    for (int i = 0; i < nbat; ++i) {
        const int buf = i % NS, tb = i & 1;
        const int ybase = ystart + i * NB;
        const bool more = i + 1 < nbat;
        // gradients of this batch from the carried rows (src/flow.cpp:225-237),
        // before any load of this iteration is issued (a fresh load sharing
        // the carried values' scoreboard would make them wait for it)
        float ctr[NB], gxs[NB], gys[NB];
#pragma unroll
        for (int b = 0; b < NB; ++b) {
            ctr[b] = cen[b + 1];
            gys[b] = 0.5f * (cen[b + 2] - cen[b]);
            float lf = __shfl_up_sync(0xffffffffu, ctr[b], 1);
            float rt = __shfl_down_sync(0xffffffffu, ctr[b], 1);
            if (lane == 0) lf = edg[b];
            if (lane == 31) rt = edg[b];
            gxs[b] = 0.5f * (rt - lf);
        }
        float nfx[NB], nfy[NB];
        if (more) {
            // next batch's taps, then the flow two batches ahead, the next
            // batch's `from` rows (ybase + NB + 1 ..) and edge neighbours
            stage_taps(ybase + NB, tb ^ 1, fl, nfx, nfy);
            const bool fl2 = i + 2 < nbat;
            cen[0] = cen[NB];
            cen[1] = cen[NB + 1];
            if (ybase + NB >= 0 && ybase + 3 * NB <= h) {  // every row below inside
                const int rb = (ybase + NB) * w;
                if (fl2) {
#pragma unroll
                    for (int b = 0; b < NB; ++b) fl[b] = Uc[rb + (NB + b) * w];
                }
#pragma unroll
                for (int j = 2; j < NB + 2; ++j) cen[j] = __ldg(Fc + (rb + (j - 1) * w));
#pragma unroll
                for (int b = 0; b < NB; ++b) edg[b] = __ldg(Fc + (rb + b * w + eoff));
            } else {
                if (fl2) {
#pragma unroll
                    for (int b = 0; b < NB; ++b) fl[b] = Uc[ro(ybase + 2 * NB + b)];
                }
#pragma unroll
                for (int j = 2; j < NB + 2; ++j) cen[j] = __ldg(Fc + ro(ybase + NB - 1 + j));
#pragma unroll
                for (int b = 0; b < NB; ++b) edg[b] = __ldg(Fc + ro(ybase + NB + b) + eoff);
            }
#ifdef FS_CHECKS
            if (g_fs_inject != 2)
#endif
                cp_async_wait<1>();
        } else {
#ifdef FS_CHECKS
            if (g_fs_inject != 2)
#endif
                cp_async_wait<0>();
        }
        float dts[NB];
#pragma unroll
        for (int b = 0; b < NB; ++b) {  // float bilinear (lerp form) of the staged taps
            const float* tp = tapb + ((tb * NB + b) * 4) * IW + c;
            const float t00 = tp[0], t10 = tp[IW], t01 = tp[2 * IW], t11 = tp[3 * IW];
#ifdef FS_CHECKS
            {  // the cp.async copies of this batch landed (wait_group) and are this batch's
                const int* ct = chk_tap + (((tb * NB + b) * IW) + c) * 3;
                const float* g = T + ct[0];
                FS_DCHECK(__float_as_int(t00) == __float_as_int(__ldg(g)) &&
                          __float_as_int(t10) == __float_as_int(__ldg(g + ct[1])) &&
                          __float_as_int(t01) == __float_as_int(__ldg(g + ct[2])) &&
                          __float_as_int(t11) == __float_as_int(__ldg(g + ct[2] + ct[1])));
            }
#endif
            const float u = __fmaf_rn(tfx[b], t10 - t00, t00);
            const float v = __fmaf_rn(tfx[b], t11 - t01, t01);
            dts[b] = __fmaf_rn(tfy[b], v - u, u) - ctr[b];
        }
        if (i >= NS) bar_sync<NT>(1 + NS + buf);  // consumers released this buffer
#ifdef FS_CHECKS
        if (i >= NS) FS_DCHECK(chk[8 + buf] == i - NS);
#endif
        float* st = stage + (size_t)buf * lk_stage_elems<M>() + c;
#pragma unroll
        for (int b = 0; b < NB; ++b) {
            const bool in = xin && (unsigned)(ybase + b) < yhi;
            const float px = in ? gxs[b] * dts[b] : 0.f, py = in ? gys[b] * dts[b] : 0.f;
            const float2 o = *rp;
            *rp = make_float2(px, py);
            V0 = (V0 + px) - o.x;
            V1 = (V1 + py) - o.y;
            rp += IW;
            if (rp == rend) rp = ring + c;
            st[b * IWP] = V0;
            st[NB * IWP + b * IWP] = V1;
#ifdef FS_CHECKS
            FS_DCHECK(rp >= ring + c && rp < rend);
#endif
        }
#ifdef FS_CHECKS
        if (c == 0) chk[buf] = i + (g_fs_inject == 1);
#endif
        bar_arrive<NT>(1 + buf);  // batch staged
        if (more) {
#pragma unroll
            for (int b = 0; b < NB; ++b) {
                tfx[b] = nfx[b];
                tfy[b] = nfy[b];
            }
        }
    }
}

// ---- consumer (fp32 later iterations): horizontal sums by row prefix sums -
// Consumer warp b takes batch row b: an exclusive-scan of the row's 128
// staged column sums (a float4 per lane, then a warp scan of the lane
// totals), written back in place; output column j's (2r+1)-wide sum is then
// P[j + 2r] - P[j - 1].  Lane l owns output columns l, l + 32, l + 64, l + 96,
// so the flow / coefficient loads and the flow stores are coalesced.
template <int M>
__device__ __forceinline__ void lk_consume_scan(const LkArgs& a, const LkDir& D, float* stage,
                                                int x0, int y0, int ystart, int yo_end,
                                                int nbat) {
    using Cfg = LkCfg<M>;
    constexpr int NB = Cfg::NB, IW = Cfg::IW, NT = Cfg::THREADS, NS = Cfg::NS;
    constexpr int CPL = IW / 32;  // staged columns per lane (consecutive)
    static_assert(NB == 4 && NT == IW + 32 * NB && CPL % 4 == 0, "one consumer warp per row");
    constexpr bool FIRST = M == LK_FIRST;
    constexpr int IWP = lk_iwp<M>(), QS = NB * IWP;
    const int r = a.r, w = a.w, tw = a.tw;
    const int t = threadIdx.x - IW;
    const int b = t >> 5, lane = t & 31;
    const int nact = min(tw, w - x0);  // output columns of this tile
    for (int i = 0; i < nbat; ++i) {
        const int buf = i % NS;
        const int yo = ystart + i * NB + b - r;
        const bool rowact = yo >= y0 && yo < yo_end;  // warp-uniform
        // lane's outputs: row yo, columns x0 + lane + 32 k (immediate offsets)
        const size_t ro = (size_t)yo * w + x0 + lane;
        const float2* __restrict__ fin = D.fin + ro;
        const float4* __restrict__ cfp = D.coef + ro;
        // CPL == 4: the row's flow / ok / coefficients prefetched before the wait
        float2 pfo[4];
        float4 pcf[4];
        uint8_t pok[4];
        if (CPL == 4 && rowact) {
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                if (lane + 32 * k < nact) {
                    pfo[k] = fin[32 * k];
                    pcf[k] = cfp[32 * k];
                    if (FIRST) pok[k] = D.okin[ro + 32 * k];
                }
            }
        }
        bar_sync<NT>(1 + buf);
#ifdef FS_CHECKS
        extern __shared__ __align__(16) unsigned char smem[];
        int* chk = reinterpret_cast<int*>(smem + lk_check_off<M>(a.r));
        FS_DCHECK(chk[buf] == i);
#endif
        if (rowact) {
            float* vb = stage + (size_t)buf * lk_stage_elems<M>() + b * IWP;
            float H[2][CPL];
#pragma unroll
            for (int q = 0; q < 2; ++q) {
                float4 v[CPL / 4];
#pragma unroll
                for (int u = 0; u < CPL / 4; ++u)
                    v[u] = *reinterpret_cast<const float4*>(vb + q * QS + CPL * lane + 4 * u);
                float run = 0.f;
#pragma unroll
                for (int u = 0; u < CPL / 4; ++u) {
                    v[u].x += run;
                    v[u].y += v[u].x;
                    v[u].z += v[u].y;
                    v[u].w += v[u].z;
                    run = v[u].w;
                }
                float s = run;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const float n = __shfl_up_sync(0xffffffffu, s, o);
                    if (lane >= o) s += n;
                }
                float ex = __shfl_up_sync(0xffffffffu, s, 1);
                if (lane == 0) ex = 0.f;
#pragma unroll
                for (int u = 0; u < CPL / 4; ++u) {
                    v[u].x += ex;
                    v[u].y += ex;
                    v[u].z += ex;
                    v[u].w += ex;
                    *reinterpret_cast<float4*>(vb + q * QS + CPL * lane + 4 * u) = v[u];
                }
                __syncwarp();
#pragma unroll
                for (int k = 0; k < CPL; ++k) {
                    const int j = lane + 32 * k;
                    if (j < tw) {
                        const float hi = vb[q * QS + j + 2 * r];
                        H[q][k] = j > 0 ? hi - vb[q * QS + j - 1] : hi;
                    }
                }
            }
            // the outputs in groups of 4 columns: the group's flow / ok /
            // coefficient loads in flight together, then solve and store
#pragma unroll
            for (int k0 = 0; k0 < CPL; k0 += 4) {
                float2 fo[4];
                float4 cf[4];
                uint8_t okv[4];
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const int j = lane + 32 * (k0 + k);
                    if (CPL == 4) {
                        fo[k] = pfo[k];
                        cf[k] = pcf[k];
                        okv[k] = pok[k];
                    } else if (j < nact) {
                        fo[k] = fin[j - lane];
                        cf[k] = cfp[j - lane];
                        if (FIRST) okv[k] = D.okin[ro + j - lane];
                    }
                }
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const int j = lane + 32 * (k0 + k);
                    if (j >= nact) continue;
                    const size_t oi = ro + (j - lane);
                    float2 f = fo[k];
                    if (FIRST) D.okout[oi] = (okv[k] || cf[k].w != 0.f) ? 1 : 0;
                    if (cf[k].w != 0.f) {  // -(M^-1 b) in float
                        const float bx = H[0][k0 + k], by = H[1][k0 + k];
                        float ndx = f.x + -__fmaf_rn(cf[k].x, bx, -(cf[k].y * by));
                        float ndy = f.y + -__fmaf_rn(cf[k].z, by, -(cf[k].y * bx));
                        final_cap(a.flow_cap, ndx, ndy);  // src/flow.cpp:283-287
                        f = make_float2(ndx, ndy);
                    }
#ifdef FS_CHECKS
                    FS_DCHECK(oi < (size_t)a.w * a.h && yo >= 0 && yo < a.h);
#endif
                    D.fout[oi] = f;
                }
            }
        }
#ifdef FS_CHECKS
        if (t == 0) chk[8 + buf] = i;
#endif
        if (i + NS < nbat) bar_arrive<NT>(1 + NS + buf);  // buffer free for batch i + NS
    }
}

// ---- consumer: horizontal sums, solve, update, next It ---------------------
template <int M>
__device__ __forceinline__ void lk_consume(const LkArgs& a, const LkDir& D,
                                           const typename LkCfg<M>::Acc* stage, int x0, int y0,
                                           int ystart, int yo_end, int nbat) {
    using Cfg = LkCfg<M>;
    using Acc = typename Cfg::Acc;
    constexpr int NB = Cfg::NB, NQ = Cfg::NQ, S = Cfg::S;
    constexpr bool FULL = Cfg::FULL, TENSOR = M == LK_TENSOR, FIRST = M == LK_FIRST;
    const int r = a.r, w = a.w;
    constexpr int IWP = lk_iwp<M>();
    const int nruns = (a.tw + S - 1) / S;
    constexpr int NT = Cfg::THREADS;
    const int t = threadIdx.x - Cfg::IW;
    const int b = t % NB, run = t / NB;  // NB * nruns <= 128 by construction
    const int cs = run * S;
    for (int i = 0; i < nbat; ++i) {
        const int buf = i & 1;
        const int yo = ystart + i * NB + b - r;
        const bool active = run < nruns && yo >= y0 && yo < yo_end && x0 + cs < w;
        const int nout = active ? min(min(S, a.tw - cs), w - (x0 + cs)) : 0;
        // prefetch the run's own flow / ok / coefficients before waiting
        float2 fo[S];
        float4 cf[S];
        uint8_t okv[S];
        if (active && !TENSOR) {
#pragma unroll
            for (int o = 0; o < S; ++o) {
                const int oi = yo * w + min(x0 + cs + o, w - 1);
                fo[o] = D.fin[oi];
                if (FULL || FIRST) okv[o] = D.okin[oi];
                if (!FULL) cf[o] = D.coef[oi];
            }
        }
        bar_sync<NT>(1 + buf);
#ifdef FS_CHECKS
        extern __shared__ __align__(16) unsigned char smem[];
        int* chk = reinterpret_cast<int*>(smem + lk_check_off<M>(a.r));
        FS_DCHECK(chk[buf] == i);
#endif
        if (active) {
            const Acc* vb = stage + (size_t)buf * lk_stage_elems<M>() + b * IWP + cs;
            const int QS = NB * IWP;  // plane stride
            Acc s[NQ], s2[NQ];
#pragma unroll
            for (int q = 0; q < NQ; ++q) s[q] = s2[q] = 0.0;
            int k = 0;
            for (; k + 1 <= 2 * r; k += 2) {  // two accumulators, no single chain
#pragma unroll
                for (int q = 0; q < NQ; ++q) {
                    s[q] += vb[q * QS + k];
                    s2[q] += vb[q * QS + k + 1];
                }
            }
            if (k <= 2 * r) {
#pragma unroll
                for (int q = 0; q < NQ; ++q) s[q] += vb[q * QS + k];
            }
#pragma unroll
            for (int q = 0; q < NQ; ++q) s[q] += s2[q];
            const Acc* va = vb + 2 * r;  // column entering the window at o
#pragma unroll
            for (int o = 0; o < S; ++o) {
                if (o >= nout) break;
                if (o > 0) {
#pragma unroll
                    for (int q = 0; q < NQ; ++q)
                        s[q] = (s[q] + va[q * QS + o]) - vb[q * QS + o - 1];
                }
                const int oi = yo * w + (x0 + cs + o);
                if (TENSOR) {  // the level's eigenvalue test and inverse tensor
                    double inv_det;
                    float4 coef = make_float4(0.f, 0.f, 0.f, 0.f);
                    if (lk_tensor_ok(s[0], s[1], s[2], a.eig_thresh, inv_det))
                        coef = make_float4((float)(s[2] * inv_det), (float)(s[1] * inv_det),
                                           (float)(s[0] * inv_det), 1.f);
                    D.coef[oi] = coef;
                    continue;
                }
                float2 f = fo[o];
                if (FIRST) D.okout[oi] = (okv[o] || cf[o].w != 0.f) ? 1 : 0;
                if (FULL) {
                    uint8_t ok = okv[o];
                    const double A = s[0], B = s[1], Cc = s[2];
                    float4 coef = make_float4(0.f, 0.f, 0.f, 0.f);
                    double inv_det;
                    if (lk_solve(A, B, Cc, s[3], s[4], a.eig_thresh, a.flow_cap, f.x, f.y,
                                     inv_det)) {
                        ok = 1;
                        coef = make_float4((float)(Cc * inv_det), (float)(B * inv_det),
                                           (float)(A * inv_det), 1.f);
                    }
                    D.okout[oi] = ok;
                    if (D.coef) D.coef[oi] = coef;
                } else if (cf[o].w != 0.f) {
                    float ndx, ndy;
                    if (Cfg::F32) {  // -(M^-1 b) in float
                        const float bx = s[0], by = s[1];
                        ndx = f.x + -__fmaf_rn(cf[o].x, bx, -(cf[o].y * by));
                        ndy = f.y + -__fmaf_rn(cf[o].z, by, -(cf[o].y * bx));
                    } else {
                        const double bx = s[0], by = s[1];
                        const double ux = -((double)cf[o].x * bx - (double)cf[o].y * by);
                        const double uy = -((double)cf[o].z * by - (double)cf[o].y * bx);
                        ndx = f.x + (float)ux;
                        ndy = f.y + (float)uy;
                    }
                    final_cap(a.flow_cap, ndx, ndy);  // src/flow.cpp:283-287
                    f = make_float2(ndx, ndy);
                }
                fo[o] = f;
                D.fout[oi] = f;
            }
        }
#ifdef FS_CHECKS
        if (t == 0) chk[8 + buf] = i;
#endif
        if (i + 2 < nbat) bar_arrive<NT>(3 + buf);  // buffer free for batch i + 2
    }
}

template <int M>
__host__ __device__ inline size_t lk_check_off(int r) {
    return lk_ring_bytes<M>(r) +
           LkCfg<M>::NS * lk_stage_elems<M>() * sizeof(typename LkCfg<M>::Acc) +
           lk_tap_bytes<M>();
}

// CERT: the row/column tiles' tap certificate (fp32 sweeps only)
template <int M, bool CERT = false>
__global__ void __launch_bounds__(LkCfg<M>::THREADS, LkCfg<M>::MINB) k_lk_sweep(LkArgs a) {
    extern __shared__ __align__(16) unsigned char smem[];
    void* ring = smem;
    auto* stage = reinterpret_cast<typename LkCfg<M>::Acc*>(smem + lk_ring_bytes<M>(a.r));
    const LkDir& D = a.d[blockIdx.z];
    const int x0 = blockIdx.x * a.tw, y0 = blockIdx.y * a.th;
    const int yo_end = min(y0 + a.th, a.h);
    const int ystart = y0 - a.r;
    const int yend = yo_end + a.r;
    const int nbat = (yend - ystart + LkCfg<M>::NB - 1) / LkCfg<M>::NB;
    if constexpr (LkCfg<M>::F32) {
        float* tapb = reinterpret_cast<float*>(smem + lk_ring_bytes<M>(a.r) +
                                               LkCfg<M>::NS * lk_stage_elems<M>() * sizeof(float));
        if (threadIdx.x < LkCfg<M>::IW)
            lk_produce_f32<M, CERT>(a, D, static_cast<float2*>(ring), stage, tapb, x0, ystart,
                                    yend, nbat);
        else
            lk_consume_scan<M>(a, D, stage, x0, y0, ystart, yo_end, nbat);
    } else if (threadIdx.x < LkCfg<M>::IW)
        lk_produce<M>(a, D, ring, stage, x0, ystart, yend, nbat);
    else
        lk_consume<M>(a, D, stage, x0, y0, ystart, yo_end, nbat);
}

FS_CHECK_TU(lk)
void check_inject_lk(int mode) {
#ifdef FS_CHECKS
    cudaMemcpyToSymbol(g_fs_inject, &mode, sizeof mode);
#else
    (void)mode;
#endif
}

namespace launch {

// the largest dynamic shared memory any sweep mode needs at radius r
static size_t lk_smem_max(int r) {
    size_t m = lk_smem_bytes<LK_ITER>(r);
    m = std::max(m, lk_smem_bytes<LK_FULL>(r));
    m = std::max(m, lk_smem_bytes<LK_TENSOR>(r));
    m = std::max(m, lk_smem_bytes<LK_FIRST>(r));
    return m;
}
static int lk_optin_bytes() {
    int dev = 0, optin = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) !=
        cudaSuccess)
        optin = 227 * 1024;  // sm_100
    return optin;
}
static std::atomic<unsigned long long> lk_configured{0};
void lk_init() {
    once_per_device(lk_configured, [](int) {
        const int mx = lk_optin_bytes();
        cudaFuncSetAttribute(k_lk_sweep<LK_ITER>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
        cudaFuncSetAttribute(k_lk_sweep<LK_FULL>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
        cudaFuncSetAttribute(k_lk_sweep<LK_TENSOR>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             mx);
        cudaFuncSetAttribute(k_lk_sweep<LK_FIRST>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             mx);
        cudaFuncSetAttribute(k_lk_sweep<LK_ITER, true>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
        cudaFuncSetAttribute(k_lk_sweep<LK_FIRST, true>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
    });
}

#ifndef LK_TH_MIN
#define LK_TH_MIN 16  // smallest tile height (smaller: faster alone, slower in the DAG)
#endif
static int lk_tile_rows(int w, int h, int r, int ndir, int per_sm, int tw, int slot_div) {
    // A CTA sweeps th + 2r rows; CTAs run in waves of 148 SMs x per_sm.  Pick th
    // minimising waves x rows per CTA (wave quantisation vs. halo rows).
    const long cols = (w + tw - 1) / tw;
    const long slots = 148L * per_sm / std::max(1, slot_div);
    int best = LK_TH_MIN;
    long best_cost = -1;
    for (int th = LK_TH_MIN; th <= 256; th += (th < 32 ? 4 : 8)) {
        const long ctas = cols * ((h + th - 1) / th) * ndir;
        const long cost = ((ctas + slots - 1) / slots) * (th + 2 * r);
        if (best_cost < 0 || cost < best_cost) {
            best_cost = cost;
            best = th;
        }
        if (th >= h) break;
    }
    return best;
}

cudaError_t lk_prep(const LkArgs& a, cudaStream_t s) {
    dim3 g((a.w + 31) / 32, (a.h + 8 * LK_PREP_ROWS - 1) / (8 * LK_PREP_ROWS), a.ndir);
    if (a.mode == 2)
        k_lk_prep<2><<<g, 256, 0, s>>>(a);
    else
        k_lk_prep<0><<<g, 256, 0, s>>>(a);
    return cudaGetLastError();
}

template <int M>
static void sweep_launch(LkArgs a, cudaStream_t s) {
    a.tw = LkCfg<M>::IW - 2 * a.r;
    if (a.th <= 0) a.th = lk_tile_rows(a.w, a.h, a.r, a.ndir, LkCfg<M>::MINB, a.tw, a.slot_div);
    dim3 g((a.w + a.tw - 1) / a.tw, (a.h + a.th - 1) / a.th, a.ndir);
    if constexpr (LkCfg<M>::F32) {
        if (a.cert_fail) {
            k_lk_sweep<M, true><<<g, LkCfg<M>::THREADS, lk_smem_bytes<M>(a.r), s>>>(a);
            return;
        }
    }
    k_lk_sweep<M><<<g, LkCfg<M>::THREADS, lk_smem_bytes<M>(a.r), s>>>(a);
}

cudaError_t lk_sweep(const LkArgs& a0, int mode, cudaStream_t s) {
    LkArgs a = a0;
    lk_init();
    switch (mode) {
        case LK_FULL: sweep_launch<LK_FULL>(a, s); break;
        case LK_TENSOR: sweep_launch<LK_TENSOR>(a, s); break;
        case LK_FIRST: sweep_launch<LK_FIRST>(a, s); break;
        default: sweep_launch<LK_ITER>(a, s); break;
    }
    return cudaGetLastError();
}

// NB * nruns must fit the 128 consumer threads: tw = 128 - 2r, runs of 4
// (FULL, NB = 4) or 8 (NB = 8) => any r <= 48 keeps tw >= 32; and every
// sweep mode's ring + staging must fit the device's shared-memory opt-in
// (r <= 45 on sm_100's 227 KB).
int lk_max_radius() {
    const size_t optin = (size_t)lk_optin_bytes();
    int r = 48;
    while (r > 1 && lk_smem_max(r) > optin) --r;
    return r;
}

}  // namespace launch
}  // namespace fs
