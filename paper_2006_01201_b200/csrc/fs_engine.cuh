// Host-side orchestration of the B200 flow+blend path: the pyramidal flow
// driver (src/flow.cpp:194-314), the fold step (src/pipeline.cpp:153-207) and
// the planned, graph-captured fold.  Internal C++ API; the boundary is the
// C-ABI in include/fs_b200.h.
#pragma once

#include <cuda_runtime.h>

#include <functional>
#include <string>
#include <vector>

#include "../../include/fs_b200.h"
#include "fs_device.cuh"

namespace fs {

struct Error {
    fs_status code;
    std::string msg;
};
[[noreturn]] void raise(fs_status code, const std::string& msg);
std::string& last_error_slot();  // thread-local message behind fs_last_error()
void cuda_check(cudaError_t e, const char* what);
#define FS_CK(x) ::fs::cuda_check((x), #x)

void validate_flow_params(const fs_flow_params& p);    // src/flow.cpp:15-21
void validate_blend_params(const fs_blend_params& p);  // src/blender.cpp:11-16
int pyramid_depth(int w, int h, int levels);           // src/flow.cpp:178-185
void ensure_device();                                  // throws FS_ERR_CUDA without sm_100
// Squared distances are int32 with the "no seed" sentinel kInfSq = 2^30 - 1:
// every in-canvas squared distance (w-1)^2 + (h-1)^2 must stay below it
// (e.g. 16384 x 16384 is fine, 32768 x 1 is not) -> FS_ERR_UNSUPPORTED.
void check_edt_extent(long long w, long long h, const char* what);

// Per-launch kernel timing (fs_plan_profile): when a profile run installs a
// KernelProf, every launch site records CUDA events around its kernel on the
// launching stream plus the launch's algorithmic bytes.
struct KernelProf {
    struct Rec {
        const char* name;
        double bytes;
        cudaEvent_t a, b;
    };
    std::vector<Rec> recs;
    ~KernelProf();
};
KernelProf*& kernel_prof();  // thread-local; nullptr = profiling off
struct ProfScope {
    cudaStream_t s;
    bool on;
    ProfScope(const char* name, double bytes, cudaStream_t s);
    ~ProfScope();
};

// Bump allocator: run the layout once with base == nullptr to size it, then
// again over one device allocation.
struct Arena {
    char* base = nullptr;
    size_t off = 0;
    template <class T>
    T* take(size_t count) {
        off = (off + 255) & ~size_t(255);
        T* p = base ? reinterpret_cast<T*>(base + off) : nullptr;
        off += count * sizeof(T);
        return p;
    }
};

struct Level {
    int w, h;
};

// A tile's tap certificate for one sweep launch (see FlowTile).
struct TileCert {
    int zlo = 0, zhi = 0, exlo = 0, exhi = 0;  // level-local, along the axis
};
// Workspace of one (bi)directional pyramidal LK problem on a w x h crop.
struct FlowWS {
    int w = 0, h = 0, depth = 0, ndir = 0;
    std::vector<Level> lv;
    std::vector<float*> pyr[2];  // level pointers (level 0 = caller's gray buffers)
    float2* fb[2][2] = {};       // [dir][pingpong] level flow
    uint8_t* ok[2][2] = {};
    std::vector<float4*> coef[2];  // [dir][level] level-constant inverse structure tensor
    // split schedule (flow_split_events): every level's structure tensor on a
    // side stream right after the pyramid, off the coarse-to-fine chain
    cudaEvent_t ev_fork = nullptr;
    std::vector<cudaEvent_t> ev_tensor;
    // a tile of a larger crop (FlowTile): the whole crop's level dims (the
    // flow caps of src/flow.cpp:241, 300-313) and the per-launch tap
    // certificates ([level * iterations + iteration])
    std::vector<Level> cap_lv;
    std::vector<TileCert> cert;
    int cert_axis = 0;
    unsigned int* cert_fail = nullptr;
    // schedule marks (fs_plan_timeline_graph): called at every level start
    // ("L<l>") and after the last level ("flow_end") on the chain's stream
    std::function<void(const std::string&, cudaStream_t)> mark;
    // split schedule: the coarsest level's tensor on the chain's own stream
    // (set by the plan for folds that start with others: on the tensor
    // stream it waited behind their side work, C2 3.381 -> 3.367 ms; a fold
    // alone, C1, is faster with it beside the chain, 0.354 -> 0.337 ms)
    bool tensor0_on_chain = false;
    void layout(Arena& a, int w, int h, int levels, int ndir);
};

// Row/column tile of a fold's flow: the crop's Area3 box
// is cut along its long axis into interiors; tile t computes the whole
// pyramidal LK on its region = interior + halo (its own crop, pyramid and
// flow), and its interior's flow equals the untiled one: the halo covers the
// dependency cone of every level (iterations x r + smoothing + the 2x
// upsample, plus the pyramid's clamped border at a cut), and the gathers of
// `to` are certified on the device to stay in the tile pyramid's exact part.
struct FlowTile {
    int axis = 0;            // 0: cut along x (column tiles), 1: along y (row tiles)
    Rect region, interior;   // box-relative
    float* gray[2] = {};
    FlowWS flow;
    float2* vec[2] = {};     // region-sized level-0 flow
    uint8_t* valid[2] = {};
};
// Plan the tiles of a w x h crop (box-relative) along `axis` with interiors
// of about tile_len; margin: extra exact pyramid border for the taps (px of
// level 0).  Returns false (no tiles) when tiling cannot be exact by
// construction: the axis length not divisible by 2^(depth-1), or a region
// that would not hold its cone.
bool plan_flow_tiles(int w, int h, int axis, int tile_len, int margin, const fs_flow_params& p,
                     std::vector<FlowTile>& tiles);
void layout_flow_tile(FlowTile& t, Arena& a, const fs_flow_params& p, int box_w, int box_h);
void flow_split_events(FlowWS& ws);   // create the split schedule's events
void flow_destroy_events(FlowWS& ws);
// Enqueue the whole coarse-to-fine flow on stream s.  ndir = 1: from=g0,
// to=g1.  ndir = 2: dir 0 is L->R (from g0), dir 1 is R->L (from g1).
// Outputs are the reference FlowField layouts (interleaved dx,dy + valid).
// With ts (and flow_split_events done) the structure tensors run on ts.
int flow_enqueue(FlowWS& ws, const float* g0, const float* g1, const fs_flow_params& p,
                 float2* const out_vec[2], uint8_t* const out_valid[2], cudaStream_t s,
                 cudaStream_t ts = nullptr);

// Distance-transform job layout for one seed mask of a fold.
struct EdtPlan {
    Rect W, C, E;
    int vfirst = 1;
    int e_left = 1, e_right = 1, e_top = 1, e_bottom = 1;
    int check = 0;
};
EdtPlan edt_plan(const Rect& C, const Rect& E, bool full_domain);
struct EdtWS {
    int *g = nullptr, *stack = nullptr, *out = nullptr;
    unsigned long long* bits = nullptr;
    void layout(Arena& a, const Rect& C, const Rect& E);  // sized for the full domain E
};

// One fold (pano = L, view k = R) on a planned Area3 box.
template <class V>
struct FoldWS {
    Rect box, E1, E2;
    EdtPlan ep[2];
    bool full_domain = false;
    int depth = 0;
    float* gray[2] = {};
    FlowWS flow;
    float2* fvec[2] = {};
    uint8_t* fvalid[2] = {};
    EdtWS edt[2];
    float4* blended = nullptr;
    float2* wgray = nullptr;  // (optional) gray of the warped constituents on Area3, box-indexed
    // row/column tiles of the flow (fs_plan_set_tiling); tiles_on cleared when
    // a tile's certificate fails (the fold then runs untiled)
    std::vector<FlowTile> tiles;
    bool tiles_on = false;
    FoldStats* st = nullptr;
    void layout(Arena& a, const Rect& box, const Rect& pano_bbox, const Rect& view_rect,
                const fs_flow_params& fp);
    void replan_edt();
};
// init the fold's statistics + partition (P: the pano's validity before the fold)
template <class V, class P>
int fold_enqueue_pre(FoldWS<V>& f, const P& pano, const V& view, cudaStream_t s);
// check box, crop+gray (L from crop_src), pyramid, flow (both directions),
// distance transforms (seed masks from `pano`'s validity).  With `es` (and
// two events) the distance transforms run on es, concurrently with the flow,
// and s waits for them at the end; with_edt = false leaves them to the caller.
template <class V, class P, class PC>
int fold_enqueue_flow_edt(FoldWS<V>& f, const P& pano, const PC& crop_src, const V& view, int ch,
                          const fs_flow_params& fp, cudaStream_t s, cudaEvent_t ev_flow0,
                          cudaEvent_t ev_flow1, cudaStream_t es = nullptr,
                          cudaEvent_t ev_fork = nullptr, cudaEvent_t ev_join = nullptr,
                          bool with_edt = true, cudaStream_t ts = nullptr,
                          cudaEvent_t ev_data = nullptr);  // s waits for it before the crop
template <class V, class P>
int fold_enqueue_edt(FoldWS<V>& f, const P& pano, const V& view, cudaStream_t s);
// Code 1 blend on Area3 + composition of the view onto the canvas
// (owner != nullptr: the planned DAG — the panorama's validity is owner <
// fold and only the Area3 box is written, with its RGBA8 values into `out`;
// the fold's Area2 copy is the caller's, launch::compose_area2)
template <class V>
int fold_enqueue_blend(FoldWS<V>& f, const Canvas& cv, const V& view, CanvasCount* cc,
                       const fs_blend_params& bp, cudaStream_t s, const uint8_t* owner = nullptr,
                       int fold = 0, uchar4* out = nullptr, const ReachCheck* rc = nullptr,
                       const PanoViews* first_cover = nullptr, bool write_cv = true);

void init_stats(FoldStats* st, cudaStream_t s);
void init_count(CanvasCount* cc, cudaStream_t s);

}  // namespace fs
