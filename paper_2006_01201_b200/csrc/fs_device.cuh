// Device-side data types and kernel declarations of the B200 flow+blend path.
#pragma once

#include <cuda_runtime.h>
#include <atomic>
#include <cstdint>
#include <cstdio>
#include <mutex>

#include "fs_math.cuh"

namespace fs {

// Run `fn` once per CUDA device (the current one) and per `flags` word:
// kernel attributes such as the dynamic shared-memory opt-in belong to a
// device's context, so a process driving several GPUs (or several threads)
// must apply them for each device, exactly once.
template <class F>
inline void once_per_device(std::atomic<unsigned long long>& flags, F&& fn) {
    int dev = 0;
    cudaGetDevice(&dev);
    const unsigned long long bit = 1ull << (dev & 63);
    if (flags.load(std::memory_order_acquire) & bit) return;
    static std::mutex mu;
    std::lock_guard<std::mutex> lock(mu);
    if (flags.load(std::memory_order_relaxed) & bit) return;
    fn(dev);
    flags.fetch_or(bit, std::memory_order_release);
}

constexpr int kInfSq = 0x3fffffff;  // "no seed" squared distance (exceeds any canvas d^2)

// ---- FS_CHECKS builds (tools/checks.sh) ------------------------------------
// compute-sanitizer is closed on this GPU pool, so the risky hand-offs carry
// their own checks in a checks build: FS_DCHECK(cond) counts violations in a
// per-translation-unit device counter (no relocatable device code needed) and
// prints the first few with their source line; fs_debug_check_failures()
// (fs_capi.cu) sums the counters.  Without FS_CHECKS every check compiles away.
#ifdef FS_CHECKS
static __device__ unsigned int g_fs_check_fail;
#define FS_DCHECK(cond)                                                                 \
    do {                                                                                \
        if (!(cond)) {                                                                  \
            if (atomicAdd(&::fs::g_fs_check_fail, 1u) < 8)                               \
                printf("FS_DCHECK failed: %s:%d %s\n", __FILE__, __LINE__, #cond);       \
        }                                                                               \
    } while (0)
// the TU's counter (defined once per .cu with FS_CHECK_TU(name))
#define FS_CHECK_TU(name)                                                               \
    unsigned int check_failures_##name(bool reset) {                                    \
        unsigned int v = 0;                                                             \
        cudaMemcpyFromSymbol(&v, g_fs_check_fail, sizeof v);                            \
        if (reset) {                                                                    \
            unsigned int z = 0;                                                         \
            cudaMemcpyToSymbol(g_fs_check_fail, &z, sizeof z);                          \
        }                                                                               \
        return v;                                                                       \
    }
#else
#define FS_DCHECK(cond) \
    do {                \
    } while (0)
#define FS_CHECK_TU(name) \
    unsigned int check_failures_##name(bool) { return 0; }
#endif
unsigned int check_failures_lk(bool reset);
unsigned int check_failures_kernels(bool reset);
unsigned int check_failures_plan(bool reset);
void check_inject_lk(int mode);

struct Rect {
    int x0 = 0, y0 = 0, w = 0, h = 0;
    __host__ __device__ int x1() const { return x0 + w; }
    __host__ __device__ int y1() const { return y0 + h; }
    __host__ __device__ bool contains(int x, int y) const {
        return x >= x0 && y >= y0 && x < x0 + w && y < y0 + h;
    }
    __host__ __device__ long long area() const { return (long long)w * h; }
};

// The running panorama: RGB in float4 (w unused), validity in its own plane.
// Pixel values of invalid pixels are undefined; every reader masks by valid.
struct Canvas {
    float4* rgb;
    uint8_t* valid;
    int w, h, ch;
};

// (float)b of a byte without the conversion pipe: 2^23 + b is a float's
// bits with b in the low mantissa byte (exact), minus 2^23.
__device__ __forceinline__ float u8f(unsigned int word, int byte) {
    return __uint_as_float(__byte_perm(word, 0x4B000000u, 0x7440u | byte)) - 8388608.f;
}

// A placed view in 8-bit RGBA (alpha >= 128 is valid, src/image.cpp:38-39),
// value = byte * (1/255) exactly as load_image (src/image.cpp:31-37).
struct ViewU8 {
    const uchar4* px;
    Rect rect;  // canvas placement
    // every pixel valid (a plan's RGB8 host views: alpha preset to 255), so
    // validity is the placement alone and needs no load
    int all_valid = 0;
    __device__ __forceinline__ bool valid_at(int x, int y) const {
        if (!rect.contains(x, y)) return false;
        if (all_valid) return true;
        return px[(size_t)(y - rect.y0) * rect.w + (x - rect.x0)].w >= 128;
    }
    __device__ __forceinline__ float4 value_at(int x, int y) const {
        const unsigned int p =
            reinterpret_cast<const unsigned int*>(px)[(size_t)(y - rect.y0) * rect.w + (x - rect.x0)];
        const float s = 1.0f / 255.0f;
        return make_float4(u8f(p, 0) * s, u8f(p, 1) * s, u8f(p, 2) * s, 0.f);
    }
};

// A placed view in float (ImageBuf semantics): float4 rgb + u8 valid.
struct ViewF4 {
    const float4* px;
    const uint8_t* valid;
    Rect rect;
    __device__ __forceinline__ bool valid_at(int x, int y) const {
        if (!rect.contains(x, y)) return false;
        return valid[(size_t)(y - rect.y0) * rect.w + (x - rect.x0)] != 0;
    }
    __device__ __forceinline__ float4 value_at(int x, int y) const {
        return px[(size_t)(y - rect.y0) * rect.w + (x - rect.x0)];
    }
};

// Validity (and value) of the panorama before a fold, read from the canvas.
struct PanoPlane {
    const uint8_t* valid;
    const float4* rgb;
    int w;
    __device__ __forceinline__ bool valid_at(int x, int y) const {
        return valid[(size_t)y * w + x] != 0;
    }
    __device__ __forceinline__ float4 value_at(int x, int y) const {
        return rgb[(size_t)y * w + x];
    }
};

// The same, derived from the views folded so far: the panorama's validity is
// the union of their masks (src/pipeline.cpp:201-204), and a pixel that no
// earlier fold blended holds the value of the first view that covered it
// (Area2 copies R, src/blender.cpp:69-71).  Lets a fold's partition, distance
// transforms and (when its Area3 box is disjoint from every earlier one) its
// L crop run without waiting for the earlier folds.  `owner` holds, per
// canvas pixel, the index of the first view covering it (0xFF: none; views
// are claimed in fold order as they arrive), so the union test is one byte.
constexpr int kMaxDagViews = 16;
struct PanoViews {
    int n;
    ViewU8 v[kMaxDagViews];
    const uint8_t* owner;
    int w;
    __device__ __forceinline__ bool valid_at(int x, int y) const {
        return owner[(size_t)y * w + x] < n;
    }
    __device__ __forceinline__ float4 value_at(int x, int y) const {
        const int m = owner[(size_t)y * w + x];
        return m < n ? v[m].value_at(x, y) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
};

// L-crop source of a fold whose Area3 box meets earlier folds' boxes: a pixel
// covered by two or more views before fold k was blended by the last of them,
// so its value is the composed canvas (final once that fold composed — the
// fold waits for the compose of the last earlier fold whose box meets its
// own); every other valid pixel still holds its first covering view's value.
struct PanoHybrid {
    PanoViews pv;
    PanoPlane plane;
    __device__ __forceinline__ bool valid_at(int x, int y) const { return pv.valid_at(x, y); }
    __device__ __forceinline__ float4 value_at(int x, int y) const {
        const int m0 = pv.owner[(size_t)y * pv.w + x];
        if (m0 >= pv.n) return make_float4(0.f, 0.f, 0.f, 0.f);
        for (int m = m0 + 1; m < pv.n; ++m)
            if (pv.v[m].valid_at(x, y)) return plane.value_at(x, y);
        return pv.v[m0].value_at(x, y);
    }
};

// Per-fold device bookkeeping (written by the partition kernel).
struct FoldStats {
    unsigned long long pv_count;  // |pano valid| before this fold (Area1 + Area3)
    unsigned long long cnt2;  // Area2 pixels
    unsigned long long cnt3;  // Area3 pixels
    int bx0, by0, bx1, by1;   // Area3 bbox (inclusive max), init (INT_MAX, INT_MAX, -1, -1)
    unsigned int edt_fail;    // bounded-domain EDT certificate failed (bit per mask)
    unsigned int box_mismatch;
    unsigned int reach_fail;  // a blend tap read a canvas pixel this rank does not hold final
    unsigned int tile_fail;   // a flow tile's gather left its exact pyramid part
};

// Seam-sharded execution (fs_plan_shard): a fold runs on a GPU whose canvas
// holds the panorama's values before that fold only where they are known to
// be final — everything inside `allow` except the Area3 boxes listed in
// `forbid` (earlier folds' strips not received, later folds already
// composed).  The blend records a tap of L that lands elsewhere, and the
// execution is repeated unsharded (fs_plan_check).
struct ReachCheck {
    int on = 0;
    int n = 0;
    Rect allow;
    Rect forbid[kMaxDagViews];
    __device__ __forceinline__ bool ok(int x, int y) const {
        if (!allow.contains(x, y)) return false;
        for (int i = 0; i < n; ++i)
            if (forbid[i].contains(x, y)) return false;
        return true;
    }
};

struct CanvasCount {
    unsigned long long valid_count;  // |pano valid|
};

// ---- flow (per level) ----
struct LkDir {
    const float* F;        // from-level
    const float* T;        // to-level
    const float2* fin;     // level flow in (mode 1) or coarse flow (mode 2)
    const uint8_t* okin;   // level ok in (mode 1) or coarse ok (mode 2)
    float2* fout;
    uint8_t* okout;   // written by the first iteration of a level only
    float4* coef;     // level-constant (c/det, b/det, a/det, ok): written by the
                      // first iteration, read by the later ones (nullptr: unused)
};
struct LkArgs {
    LkDir d[2];
    int ndir;
    int w, h;    // level dims
    int cw, ch;  // coarse dims (mode 2)
    double sx, sy;
    int mode;    // 0 zero, 1 flow-in, 2 upsample-from-coarse
    int r;
    int tw, th;  // output tile (th <= 0: chosen per level)
    int slot_div;  // th choice: the CTA slots a launch can expect (148 x CTAs/SM / slot_div)
    double eig_thresh;
    float flow_cap;
    // row/column tiles (FlowTile): the taps of the pixels whose coordinate
    // along cert_axis lies in [zlo, zhi) must stay inside [exlo, exhi), the
    // part of the tile's pyramid equal to the whole crop's; else *cert_fail
    // is set (nullptr: no check)
    unsigned int* cert_fail;
    int cert_axis, zlo, zhi, exlo, exhi;
};

struct SmoothArgs {
    const float2* fin[2];
    float2* fout[2];
    const uint8_t* ok[2];
    uint8_t* valid_out[2];  // written when final_cap > 0 (finalisation)
    int ndir, w, h, passes;  // passes: 1 or 2
    float final_cap;         // > 0: level-0 finalisation (cap + valid)
};

// ---- distance transform ----
// Seed masks of the fold: Area1 = pano valid && !view valid, Area2 = view
// valid && !pano valid (src/blend_field.cpp:100-104 on src/image.cpp:115-132).
template <class V, class P>
struct FoldMask {
    P pano;
    V view;
    int which;  // 1 or 2
    __device__ __forceinline__ bool operator()(int x, int y) const {
        bool pv = pano.valid_at(x, y);
        bool rv = view.valid_at(x, y);
        return which == 1 ? (pv && !rv) : (rv && !pv);
    }
};
// A plain u8 mask plane (standalone distance_transform).
struct PlaneMask {
    const uint8_t* m;
    int w;
    __device__ __forceinline__ bool operator()(int x, int y) const {
        return m[(size_t)y * w + x] != 0;
    }
};

// Region-label plane compared against one label (compute_blend's m1/m2).
struct LabelMask {
    const uint8_t* label;
    int w;
    uint8_t value;
    __device__ __forceinline__ bool operator()(int x, int y) const {
        return label[(size_t)y * w + x] == value;
    }
};

template <class M>
struct EdtJob {
    M mask;
    int which = 0;   // 0 plain, 1 Area1, 2 Area2 (selects the "have" test)
    int active = 0;
    Rect W, C;       // seed domain, output box (C inside W)
    int vfirst = 1;  // 1: columns 1-D first, envelope along rows
    int* g = nullptr;           // pass-1 output, laid out line-contiguous for pass 2
    unsigned long long* bits = nullptr;  // [nseg][nlines] seed bits per 64-position segment
    int* stack = nullptr;       // [pass-2 lines][sites]
    int* out = nullptr;         // squared distance on C, row-major C.w
    int e_left = 1, e_right = 1, e_top = 1, e_bottom = 1;  // W side == seed-bbox side
    int check = 0;
};

namespace launch {
void init();     // one-time kernel attributes (call before any graph capture)
void stamp(unsigned long long* slot, cudaStream_t);  // %globaltimer (ns) into *slot
// RGB8 host formats: n RGB8 pixels -> RGBA8 (alpha 255); canvas rect -> RGB8
// (canvas-indexed: out + 3 * (y * cw + x)); `in` of expand_rgb 4-byte aligned
void expand_rgb(const uint8_t* in, uchar4* out, size_t n, cudaStream_t);
// rectangle r (view-local) of a w-wide RGB8 image -> RGBA8 (alpha 255)
void expand_rgb_rect(const uint8_t* in, uchar4* out, int w, const Rect& r, cudaStream_t);
// alpha of n RGBA8 pixels := 255 (RGB kept)
void set_alpha(uchar4* px, size_t n, cudaStream_t);
void pack_rgb(const uchar4* in, int cw, const Rect& r, uint8_t* out, cudaStream_t);
// fs_remap.cu: overlap channel sums of view k against its first covering views
void chroma_sums(const uint8_t* owner, int cw, const ViewU8& vk, const PanoViews& pv, int k,
                 unsigned long long* sums, cudaStream_t s);
// fs_remap.cu: table-driven bilinear fisheye remap with chromaticity gains
void remap_rgba8(const uint8_t* src, int sw, int sh, int channels, const float2* map, int w, int h,
                 const float g[3], uchar4* out, cudaStream_t s);
void lk_init();  // fs_lk.cu: LK kernels' shared-memory opt-in
template <class V> void union_valid(const Canvas&, const V&, cudaStream_t);
// owner[p] = k where view k is valid and no earlier view claimed p
// (hist: += the pixels claimed, at hist[k])
void claim_owner(uint8_t* owner, int w, const ViewU8& view, int k, cudaStream_t,
                 unsigned long long* hist = nullptr);
// out != nullptr: also the RGBA8 value of every valid pixel written;
// write_cv false: the float canvas is not written (the DAG's first-cover
// pixels are read from the views, blend_area3's first_cover)
template <class V>
void place_view(const Canvas&, const V&, CanvasCount*, cudaStream_t, uchar4* out = nullptr,
                bool write_cv = true);
template <class V, class P> void partition(const P&, const V&, FoldStats*, cudaStream_t);
void snapshot_count(FoldStats* st, const CanvasCount* cc, cudaStream_t);  // pv_count = cc
void check_box(FoldStats*, const Rect&, cudaStream_t);
template <class V, class P>
void crop_gray(const P&, const V&, const Rect&, int ch, float*, float*, cudaStream_t);
void downsample(const float* in0, const float* in1, float* out0, float* out1, int w, int h,
                int nimg, cudaStream_t);
cudaError_t lk_prep(const LkArgs&, cudaStream_t);              // mode 0 or 2
// one LK sweep; mode: 0 a later iteration, 1 a level's first iteration in one
// pass, 2 the level's structure tensor alone, 3 a first iteration on it
cudaError_t lk_sweep(const LkArgs&, int mode, cudaStream_t);
int lk_max_radius();
void smooth(const SmoothArgs&, cudaStream_t);
void finalize_flow(const SmoothArgs&, cudaStream_t);
template <class M>
void edt(const EdtJob<M>&, const EdtJob<M>&, const FoldStats*, cudaStream_t);
// owner != nullptr: the panorama's validity before fold `fold` is owner < fold
template <class V>
void blend_area3(const Canvas&, const V&, const Rect&, const float2*, const float2*, const int*,
                 const int*, FoldStats*, double, double, float4*, float2*,
                 const uint8_t* owner, int fold, cudaStream_t, const ReachCheck* rc = nullptr,
                 const PanoViews* first_cover = nullptr,
                 uchar4* canvas_out = nullptr);  // set: the RGBA8 canvas, not the box buffer
template <class V>
void compose_area2(const Canvas&, const V&, const uint8_t* owner, int fold, cudaStream_t,
                   uchar4* out = nullptr, const Rect* clip = nullptr,
                   const Rect* cv_clip = nullptr);  // float canvas written only inside cv_clip
// pv_count of fold k = sum of hist[m] over m < k
void count_from_hist(FoldStats* st, const unsigned long long* hist, int k, cudaStream_t);
template <class V>
void compose_area3(const Canvas&, const V&, const Rect& box, const float4*, const uint8_t* owner,
                   int fold, cudaStream_t, uchar4* out = nullptr,
                   bool write_cv = true);  // false: only `out` (no later fold reads the canvas)
template <class V>
void compose(const Canvas&, const V&, const Rect&, const float4*, CanvasCount*, const FoldStats*,
             cudaStream_t);
void quantize(const Canvas&, uchar4*, cudaStream_t);
void quantize_rect(const Canvas&, const Rect&, uchar4*, cudaStream_t);  // canvas-indexed out
void export_float(const Canvas&, float*, uint8_t*, cudaStream_t);
}  // namespace launch

}  // namespace fs
