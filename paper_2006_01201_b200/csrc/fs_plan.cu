// Planned, graph-captured fold over 8-bit views (the production path of
// include/fs_b200.h).  A plan fixes the layout and owns every device buffer;
// one execution is a single CUDA-graph launch that recomputes the whole fold
// (partition, crop+gray, pyramid, bidirectional LK, distance transforms,
// Code 1 blend, composition, 8-bit quantisation) from the views in HBM.
#include <algorithm>
#include <array>
#include <cstdio>
#include <climits>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "fs_engine.cuh"

using namespace fs;
namespace fs {
FS_CHECK_TU(plan)
}  // namespace fs

constexpr size_t kMaxStamps = 512;

// LK structure tensors off the coarse-to-fine chain (FlowWS split schedule)
#ifndef FS_LK_SPLIT
#define FS_LK_SPLIT 1  // the level tensors off the chain (TENSOR), then fp32 FIRST + ITER
#endif
constexpr bool kLkSplit = FS_LK_SPLIT != 0;
// RGB8 upload order (plan_chunks): 0 = chosen per plan (crop parts first
// when the folds bound the execution, else whole views), 1 = every fold's
// Area3 box parts first, then the rest (measured C2 e2e 5.81 vs 4.97 ms:
// the pitched copies run at ~36 GB/s and the first-cover read-backs wait
// for the late "rest" chunks), 2 = crop parts first always.
#ifndef FS_UPLOAD_BOXES
#define FS_UPLOAD_BOXES 0
#endif
constexpr bool kUploadBoxesFirst = FS_UPLOAD_BOXES == 1;

// first-cover copies a sharded rank keeps around each own fold's Area3 box:
// a blend tap farther out is refused (ReachCheck) and the panorama runs unsharded
constexpr int kShardMargin = 128;

struct fs_plan_s {
    int device = 0;
    int n = 0;
    std::vector<Rect> rects;
    int cw = 0, chh = 0;
    fs_flow_params fp{};
    fs_blend_params bp{};
    char* arena = nullptr;
    std::vector<uchar4*> views;
    uchar4* out = nullptr;
    Canvas cv{};
    CanvasCount* cc = nullptr;
    std::vector<FoldWS<ViewU8>> folds;  // fold k is folds[k-1]
    std::vector<Rect> pano_bbox;        // superset of pano valid before fold k
    cudaStream_t cap = nullptr;
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    int launches = 0;
    std::string err;
    // DAG schedule (n <= kMaxDagViews): per-fold branch streams for the
    // partition-independent work, an ordered blend/compose chain on the main
    // stream; crop_wait[k]: the last earlier fold whose Area3 box meets fold
    // k's (0: none, the L crop is read from the views alone).
    bool dag = false;
    std::vector<cudaStream_t> branch;
    std::vector<cudaEvent_t> ev_branch, ev_compose, ev_h2d, ev_own, ev_efork, ev_ejoin;
    std::vector<cudaStream_t> edt_stream;  // per fold: the distance transforms
    std::vector<cudaStream_t> tensor_stream;  // per fold: the LK structure tensors
    std::vector<cudaStream_t> a2_stream;      // per fold: the Area2 copy (host uploads)
    cudaEvent_t ev_start = nullptr, ev_place = nullptr, ev_out = nullptr;
    cudaStream_t h2d = nullptr, d2h = nullptr, own = nullptr;
    uint8_t* owner = nullptr;  // first covering view per canvas pixel (PanoViews)
    unsigned long long* hist = nullptr;  // pixels first covered by each view (claim counts)
    cudaEvent_t ev_clear = nullptr;      // canvas planes cleared (Area2 copies may write)
    FoldStats* hstats = nullptr;  // page-locked copy of the folds' statistics (fs_plan_check)
    std::vector<int> crop_wait;
    // final_rects[k]: canvas rectangles no fold after k writes (k = 0: the
    // placement of view 0).  Split by fold k's Area3 box into reads that wait
    // for fold k's compose in the chain (late) and reads that wait only for
    // the Area2 copies / composes that can touch them (early).
    std::vector<std::vector<Rect>> final_rects;
    struct Readback {
        Rect r;
        std::vector<int> a2;  // folds whose Area2 copy may write r
        int compose = 0;      // last fold whose chain compose may write r (0: none)
        bool place = false;   // view 0's placement may write r
    };
    std::vector<std::vector<Readback>> early, late;
    // canvas rectangles no view covers: zero in the RGBA8 output, written by a
    // host function inside the graph instead of crossing PCIe
    std::vector<Rect> empty_rects;
    cudaStream_t hfill = nullptr;
    cudaEvent_t ev_hfill1 = nullptr;
    uint8_t* hfill_out = nullptr;
    std::vector<Rect> boxes;  // Area3 box of fold k (k >= 1)
    std::vector<cudaEvent_t> ev_a2;  // fold k's Area2 copied
    cudaStream_t d2h_early = nullptr;
    cudaEvent_t ev_out_early = nullptr;
    // graph with the host copies inside (execute_host), keyed by the pointers
    cudaGraph_t hgraph = nullptr;
    cudaGraphExec_t hexec = nullptr;
    std::vector<const void*> hkey;
    // host formats (fs_plan_set_host_format): RGB8 views are expanded on
    // arrival, the canvas packed to RGB8 before its read-backs
    int hv_ch = 4, ho_ch = 4;
    // RGB8 views (every pixel valid, alpha preset to 255 on the device) cross
    // PCIe in chunks ordered by need: first each fold's Area3 box parts of the
    // views it crops (fold order), then the rest of every view (view order).
    // Validity needs no data, so claims, partitions and distance transforms
    // start at once; a fold's crop waits for its box chunks only.
    struct Chunk {
        int view;
        Rect r;  // canvas coordinates
    };
    std::vector<Chunk> chunks;
    bool crop_first = false;  // plan_chunks' order (see there)
    // %globaltimer when each view's last chunk was expanded: device-side
    // telemetry, and the graph node it takes keeps the copy chain flowing
    // (without one the crop-first order measured 5.1 instead of 4.0 ms, C2)
    unsigned long long* landed = nullptr;
    std::vector<int> crop_chunk;  // per fold: last chunk its crop reads (-1: none)
    std::vector<int> done_chunk;  // per view k: last chunk of views 0..k
    std::vector<cudaEvent_t> ev_chunk, ev_copied;  // expanded / landed
    // row/column flow tiles (fs_plan_set_tiling): per fold and tile a stream
    // (+ one for its structure tensors), the tile-done event and the last
    // earlier fold whose Area3 box meets the tile's region (its crop waits
    // for that compose; 0: the views alone)
    char* tile_arena = nullptr;
    int tile_len = 0, tile_margin = 0;
    std::vector<std::vector<cudaStream_t>> tile_s, tile_ts;
    std::vector<std::vector<cudaEvent_t>> ev_tile;
    std::vector<cudaEvent_t> ev_tfork;
    std::vector<std::vector<int>> tile_wait;
    cudaStream_t xst = nullptr;  // expands chunks as they land (the copy engine never waits)
    uint8_t* stage_in = nullptr;   // RGB8 views, 4-byte aligned each
    std::vector<size_t> stage_off;
    uint8_t* stage_out = nullptr;  // RGB8 canvas
    // timeline capture (fs_plan_timeline): timing events at schedule points
    bool tl = false;
    std::vector<std::pair<std::string, cudaEvent_t>> tl_marks;
    // graph timeline (fs_plan_timeline_graph): %globaltimer stamp kernels
    bool tl_stamp = false;
    unsigned long long* stamps = nullptr;
    std::vector<std::string> stamp_labels;
    // seam sharding (fs_plan_shard): this rank's segments, one graph each
    struct Shard {
        int nranks = 1, rank = 0, nseg = 1;
        std::vector<int> fold_rank, stage;
        std::vector<fs_strip_xfer> xfers;          // every rank's transfers
        std::vector<std::vector<int>> apply, own;  // per segment: strips composed, folds run
        std::vector<ReachCheck> reach;             // per fold (own folds)
        std::vector<int> wait_local;  // per fold: last same-segment local fold its crop needs
        std::vector<cudaGraph_t> graph;
        std::vector<cudaGraphExec_t> exec;
        cudaEvent_t ev_seg = nullptr;
        std::vector<int> launches;  // per segment
        std::vector<std::vector<const void*>> hkeys;  // host pointers captured, per segment
        // rank 0's read-backs per segment: [seg][0] once the segment's strips
        // are composed (segment 0: the first-cover copies), [seg][1] after its
        // own folds' composes
        std::vector<std::array<std::vector<fs_plan_s::Readback>, 2>> reads;
        cudaEvent_t ev_place0 = nullptr;  // view 0's first-cover copy on rank 0
        cudaEvent_t ev_segend = nullptr, ev_d2h = nullptr;
        Rect clip;                          // first-cover copies needed here (rank != 0)
        unsigned long long* hist = nullptr;  // owner-plane histogram (|pano valid| per fold)
        cudaEvent_t ev_hist = nullptr;
    } shard;
};

namespace {

template <class F>
fs_status plan_guard(F&& fn) {
    try {
        fn();
        return FS_OK;
    } catch (const Error& e) {
        last_error_slot() = e.msg;
        return e.code;
    }
}

Rect rect_union(const Rect& a, const Rect& b) {
    if (a.w <= 0 || a.h <= 0) return b;
    int x0 = std::min(a.x0, b.x0), y0 = std::min(a.y0, b.y0);
    int x1 = std::max(a.x1(), b.x1()), y1 = std::max(a.y1(), b.y1());
    return Rect{x0, y0, x1 - x0, y1 - y0};
}
bool rects_meet(const Rect& a, const Rect& b);
Rect rect_inter(const Rect& a, const Rect& b) {
    int x0 = std::max(a.x0, b.x0), y0 = std::max(a.y0, b.y0);
    int x1 = std::min(a.x1(), b.x1()), y1 = std::min(a.y1(), b.y1());
    return Rect{x0, y0, std::max(0, x1 - x0), std::max(0, y1 - y0)};
}

ViewU8 view_of(const fs_plan_s* p, int k) {
#ifdef FS_NO_ALL_VALID
    return ViewU8{p->views[k], p->rects[k]};
#else
    // RGB8 host views are valid everywhere (fs_plan_set_host_format)
    return ViewU8{p->views[k], p->rects[k], p->hv_ch == 3 ? 1 : 0};
#endif
}

PanoViews views_before(const fs_plan_s* p, int k) {
    PanoViews pv{};
    pv.n = k;
    for (int m = 0; m < k; ++m) pv.v[m] = view_of(p, m);
    pv.owner = p->owner;
    pv.w = p->cw;
    return pv;
}

// One view's host -> device copy in the plan's host format.
void upload_view(fs_plan_s* p, int k, const uint8_t* src, cudaStream_t st) {
    const size_t np = (size_t)p->rects[k].w * p->rects[k].h;
    if (p->hv_ch == 4) {
        FS_CK(cudaMemcpyAsync(p->views[k], src, np * 4, cudaMemcpyDefault, st));
        return;
    }
    uint8_t* stg = p->stage_in + p->stage_off[k];
    FS_CK(cudaMemcpyAsync(stg, src, np * 3, cudaMemcpyDefault, st));
    launch::expand_rgb(stg, p->views[k], np, st);
}
// Part of an RGB8 view (canvas rectangle r inside view k) host -> device:
// a pitched copy into the view's staging image on st; expand_chunk turns it
// into RGBA8 (on another stream, so the copies run back to back).
void expand_chunk(fs_plan_s* p, int k, const Rect& r, cudaStream_t st) {
    const Rect& v = p->rects[k];
    const size_t off = (size_t)(r.y0 - v.y0) * v.w;
    if (r.x0 == v.x0 && r.w == v.w && off % 4 == 0) {  // whole rows, aligned: vectorised
        launch::expand_rgb(p->stage_in + p->stage_off[k] + off * 3, p->views[k] + off,
                           (size_t)r.w * r.h, st);
        return;
    }
    launch::expand_rgb_rect(p->stage_in + p->stage_off[k], p->views[k], v.w,
                            Rect{r.x0 - v.x0, r.y0 - v.y0, r.w, r.h}, st);
}
void upload_chunk(fs_plan_s* p, int k, const Rect& r, const uint8_t* src, cudaStream_t st) {
    const Rect& v = p->rects[k];
    const Rect l{r.x0 - v.x0, r.y0 - v.y0, r.w, r.h};
    const size_t pitch = (size_t)v.w * 3, off = ((size_t)l.y0 * v.w + l.x0) * 3;
    uint8_t* stg = p->stage_in + p->stage_off[k];
    if (l.w == v.w)
        FS_CK(cudaMemcpyAsync(stg + off, src + off, pitch * l.h, cudaMemcpyDefault, st));
    else
        FS_CK(cudaMemcpy2DAsync(stg + off, pitch, src + off, pitch, (size_t)l.w * 3, l.h,
                                cudaMemcpyDefault, st));
}
// The chunk order of the RGB8 upload (fs_plan_s::chunks).
void plan_chunks(fs_plan_s* p) {
    const int n = p->n;
    std::vector<std::vector<Rect>> rem(n);
    for (int m = 0; m < n; ++m) rem[m] = {p->rects[m]};
    p->chunks.clear();
    auto carve = [&](int m, const Rect& x) {  // move rem[m] ∩ x into chunks
        std::vector<Rect> keep;
        for (const Rect& r : rem[m]) {
            const Rect i = rect_inter(r, x);
            if (i.w <= 0 || i.h <= 0) {
                keep.push_back(r);
                continue;
            }
            p->chunks.push_back({m, i});
            if (i.y0 > r.y0) keep.push_back({r.x0, r.y0, r.w, i.y0 - r.y0});
            if (i.y1() < r.y1()) keep.push_back({r.x0, i.y1(), r.w, r.y1() - i.y1()});
            if (i.x0 > r.x0) keep.push_back({r.x0, i.y0, i.x0 - r.x0, i.h});
            if (i.x1() < r.x1()) keep.push_back({i.x1(), i.y0, r.x1() - i.x1(), i.h});
        }
        rem[m] = keep;
    };
    // Crop parts first when the folds, not the link, bound the execution:
    // then the folds that start at once (their flows need only their boxes'
    // pixels) start a view's upload earlier, and the rest of every view
    // follows in view order (the blends need whole views); a view whose
    // fold's box spans whole rows of it sends those rows in its turn and the
    // rest last (C2 e2e 4.55 -> 4.03 ms).  When the link bounds it (C4: 13.3
    // vs 15.8 ms) the pitched crop-part copies only slow it down: whole views
    // in fold order.  Estimate: ~0.3 ms per Mpx of Area3 boxes on the device
    // vs the larger direction's bytes at ~50 GB/s.
    double box_mpx = 0, in_b = 0, out_b = (double)p->cw * p->chh * p->ho_ch;
    for (int k = 1; k < n; ++k) box_mpx += p->boxes[k].area() * 1e-6;
    for (int m = 0; m < n; ++m) in_b += (double)p->rects[m].area() * 3;
    p->crop_first = FS_UPLOAD_BOXES == 2 ||
                    (FS_UPLOAD_BOXES == 0 && 0.3 * box_mpx > std::max(in_b, out_b) / 50e6);
    // test hook (tests/test_gpu_parity.py): FS_UPLOAD_ORDER=crop|views forces
    // the order, so both are checked on the same layout
    if (const char* o = getenv("FS_UPLOAD_ORDER")) {
        if (!strcmp(o, "crop")) p->crop_first = true;
        if (!strcmp(o, "views")) p->crop_first = false;
    }
    if (p->crop_first) {
        for (int k = 1; k < n; ++k)
            if (!p->crop_wait[k])
                for (int m = k; m >= 0; --m) carve(m, p->boxes[k]);
        std::vector<std::pair<int, Rect>> late;
        for (int m = 0; m < n; ++m) {
            const Rect& v = p->rects[m];
            const Rect b = m >= 1 && p->crop_wait[m] ? rect_inter(v, p->boxes[m]) : Rect{};
            const bool rows = b.w == v.w && b.h > 0 && b.h < v.h;
            if (rows) carve(m, b);
            for (const Rect& r : rem[m])
                if (r.w > 0 && r.h > 0) {
                    if (rows)
                        late.push_back({m, r});
                    else
                        p->chunks.push_back({m, r});
                }
        }
        for (const auto& c : late) p->chunks.push_back({c.first, c.second});
    } else {
        if (kUploadBoxesFirst)
            for (int k = 1; k < n; ++k)
                for (int m = k; m >= 0; --m) carve(m, p->boxes[k]);
        for (int m = 0; m < n; ++m)
            for (const Rect& r : rem[m])
                if (r.w > 0 && r.h > 0) p->chunks.push_back({m, r});
    }
    const int nc = (int)p->chunks.size();
    p->crop_chunk.assign(n, -1);
    p->done_chunk.assign(n, -1);
    for (int i = 0; i < nc; ++i) {
        const auto& c = p->chunks[i];
        for (int k = std::max(1, c.view); k < n; ++k)
            if (rects_meet(c.r, p->boxes[k])) p->crop_chunk[k] = std::max(p->crop_chunk[k], i);
        for (int k = c.view; k < n; ++k) p->done_chunk[k] = std::max(p->done_chunk[k], i);
    }
    for (auto e : p->ev_chunk) cudaEventDestroy(e);
    for (auto e : p->ev_copied) cudaEventDestroy(e);
    p->ev_chunk.assign(nc, nullptr);
    p->ev_copied.assign(nc, nullptr);
    for (int i = 0; i < nc; ++i) {
        FS_CK(cudaEventCreateWithFlags(&p->ev_chunk[i], cudaEventDisableTiming));
        FS_CK(cudaEventCreateWithFlags(&p->ev_copied[i], cudaEventDisableTiming));
    }
    if (!p->xst) {  // the expansions gate the folds' crops: highest priority
        int least = 0, greatest = 0;
        FS_CK(cudaDeviceGetStreamPriorityRange(&least, &greatest));
        FS_CK(cudaStreamCreateWithPriority(&p->xst, cudaStreamNonBlocking, greatest));
    }
}

// A tile's interior flow (both directions) into its fold's box-sized planes.
void copy_tile_interior(const FoldWS<ViewU8>& f, const FlowTile& t, cudaStream_t s) {
    const Rect &I = t.interior, &R = t.region;
    const size_t so = (size_t)(I.y0 - R.y0) * R.w + (I.x0 - R.x0);
    const size_t dof = (size_t)I.y0 * f.box.w + I.x0;
    for (int d = 0; d < 2; ++d) {
        FS_CK(cudaMemcpy2DAsync(f.fvec[d] + dof, (size_t)f.box.w * sizeof(float2), t.vec[d] + so,
                                (size_t)R.w * sizeof(float2), (size_t)I.w * sizeof(float2), I.h,
                                cudaMemcpyDeviceToDevice, s));
        FS_CK(cudaMemcpy2DAsync(f.fvalid[d] + dof, f.box.w, t.valid[d] + so, R.w, I.w, I.h,
                                cudaMemcpyDeviceToDevice, s));
    }
}
Rect tile_canvas_rect(const FoldWS<ViewU8>& f, const FlowTile& t) {
    return Rect{f.box.x0 + t.region.x0, f.box.y0 + t.region.y0, t.region.w, t.region.h};
}

// A canvas rectangle device -> host in the plan's host format.
void download_rect(fs_plan_s* p, const Rect& r, uint8_t* dst, cudaStream_t st) {
    const int c = p->ho_ch;
    const uint8_t* src = reinterpret_cast<const uint8_t*>(p->out);
    if (c == 3) {
        launch::pack_rgb(p->out, p->cw, r, p->stage_out, st);
        src = p->stage_out;
    }
    const size_t pitch = (size_t)p->cw * c;
    const size_t off = (size_t)r.y0 * pitch + (size_t)r.x0 * c;
    if (r.w == p->cw)
        FS_CK(cudaMemcpyAsync(dst + off, src + off, pitch * r.h, cudaMemcpyDefault, st));
    else
        FS_CK(cudaMemcpy2DAsync(dst + off, pitch, src + off, pitch, (size_t)r.w * c, r.h,
                                cudaMemcpyDefault, st));
}

// Host buffers of one execute_host call (nullptr members: device-resident).
struct HostIO {
    const uint8_t* const* views = nullptr;
    uint8_t* out = nullptr;
};

// Host node: zero the output's rectangles no view covers (a few threads:
// ~40 GB/s on the box's host memory vs ~50 GB/s for the same bytes over PCIe,
// and concurrent with the device-to-host copies instead of queued with them).
void CUDART_CB host_fill_empty(void* arg) {
    const fs_plan_s* p = static_cast<const fs_plan_s*>(arg);
    const size_t c = (size_t)p->ho_ch;
    const size_t pitch = (size_t)p->cw * c;
    struct Band {
        uint8_t* dst;
        size_t row_bytes, rows;
    };
    std::vector<Band> bands;
    size_t total = 0;
    for (const Rect& r : p->empty_rects) {
        uint8_t* d = p->hfill_out + (size_t)r.y0 * pitch + (size_t)r.x0 * c;
        if (r.w == p->cw)
            bands.push_back({d, pitch * r.h, 1});
        else
            bands.push_back({d, (size_t)r.w * c, (size_t)r.h});
        total += (size_t)r.w * r.h * c;
    }
    auto fill = [&](size_t part, size_t nparts) {
        for (const Band& b : bands)
            for (size_t y = 0; y < b.rows; ++y) {
                // split every row (or full-width band) into nparts slices
                const size_t lo = b.row_bytes * part / nparts, hi = b.row_bytes * (part + 1) / nparts;
                if (hi > lo) std::memset(b.dst + y * (b.rows > 1 ? pitch : 0) + lo, 0, hi - lo);
            }
    };
    const size_t nthreads = total >= (64u << 20) ? 4 : 1;
    std::vector<std::thread> th;
    for (size_t t = 1; t < nthreads; ++t) th.emplace_back(fill, t, nthreads);
    fill(0, nthreads);
    for (auto& t : th) t.join();
}

// Enqueue one full execution on stream s (captured into a graph).
//
// serial (dag = false; fs_plan_profile and n > kMaxDagViews): the folds one
// after another on s, the 8-bit panorama quantised at the end.
//
// dag: fold k's partition, crop, pyramid, flow and distance transforms run on
// its own branch stream as soon as views 0..k exist (and, when its L crop
// needs the composed panorama, after fold k-1's compose); only the blend +
// compose of the folds form an ordered chain on s.  A fold's |pano valid| is
// chained from the previous fold's partition counts.  Each canvas rectangle
// is quantised (and, with io->out, copied to the host) on the d2h stream as
// soon as the last fold that writes it composed.  With io->views, the views
// are copied in fold order on the h2d stream and each fold starts when its
// views have landed — host transfers overlap the folds.
int enqueue_all(fs_plan_s* p, cudaStream_t s, bool dag, const HostIO* io = nullptr) {
    int launches = 0;
    auto mark = [&](const std::string& label, cudaStream_t st) -> cudaEvent_t {
        if (p->tl_stamp) {
            if (p->stamp_labels.size() < kMaxStamps) {
                launch::stamp(p->stamps + p->stamp_labels.size(), st);
                p->stamp_labels.push_back(label);
            }
            return nullptr;
        }
        if (!p->tl) return nullptr;
        cudaEvent_t e;
        FS_CK(cudaEventCreate(&e));
        FS_CK(cudaEventRecord(e, st));
        p->tl_marks.push_back({label, e});
        return e;
    };
    auto tl_event = [&](const std::string& label) -> cudaEvent_t {
        if (!p->tl) return nullptr;
        cudaEvent_t e;
        FS_CK(cudaEventCreate(&e));
        p->tl_marks.push_back({label, e});
        return e;
    };
    mark("t0", s);
    const PanoPlane plane{p->cv.valid, p->cv.rgb, p->cv.w};
    const bool hin = io && io->views, hout = io && io->out;
    const bool hfill = dag && hout && !p->empty_rects.empty();
    // RGB8 views in chunks (validity needs no data): ev_view[k] = views 0..k
    // complete, ev_crop[k] = fold k's crop inputs in
    const bool chunked = dag && hin && p->hv_ch == 3 && !p->chunks.empty();
    // RGB8 views (valid everywhere): the blends read a first-cover pixel of L
    // from its view, so the float canvas holds only blended pixels (the
    // placement and Area2 copies write the RGBA8 output alone)
#ifdef FS_NO_FIRST_COVER
    const bool fc_mode = false;
#else
    const bool fc_mode = dag && p->hv_ch == 3;
#endif
    const Rect no_cv{0, 0, 0, 0};
    std::vector<cudaEvent_t> ev_view(p->n, nullptr), ev_crop(p->n, nullptr);
    if (hin) {
        for (int k = 0; k < p->n; ++k) {
            ev_view[k] = chunked ? p->ev_chunk[p->done_chunk[k]] : p->ev_h2d[k];
            ev_crop[k] = chunked ? (p->crop_chunk[k] >= 0 ? p->ev_chunk[p->crop_chunk[k]] : nullptr)
                                 : p->ev_h2d[k];
        }
    }
    if (dag) {
        FS_CK(cudaEventRecord(p->ev_start, s));
        if (hfill) {  // uncovered canvas: zeroed by the host, concurrently
            p->hfill_out = io->out;
            FS_CK(cudaStreamWaitEvent(p->hfill, p->ev_start, 0));
            FS_CK(cudaLaunchHostFunc(p->hfill, host_fill_empty, p));
            FS_CK(cudaEventRecord(p->ev_hfill1, p->hfill));
        }
        if (hin) {
            FS_CK(cudaStreamWaitEvent(p->h2d, p->ev_start, 0));
            if (chunked) {
                int next = 0;  // next view whose completion to mark
                FS_CK(cudaStreamWaitEvent(p->xst, p->ev_start, 0));
                for (int i = 0; i < (int)p->chunks.size(); ++i) {
                    const auto& c = p->chunks[i];
                    upload_chunk(p, c.view, c.r, io->views[c.view], p->h2d);
                    FS_CK(cudaEventRecord(p->ev_copied[i], p->h2d));
                    FS_CK(cudaStreamWaitEvent(p->xst, p->ev_copied[i], 0));
                    expand_chunk(p, c.view, c.r, p->xst);
                    FS_CK(cudaEventRecord(p->ev_chunk[i], p->xst));
                    while (next < p->n && p->done_chunk[next] == i) {
                        launch::stamp(p->landed + next, p->xst);
                        mark("h2d_" + std::to_string(next++), p->xst);
                    }
                }
                FS_CK(cudaEventRecord(p->ev_h2d[p->n - 1], p->xst));  // joined at the end
            } else {
                for (int k = 0; k < p->n; ++k) {
                    upload_view(p, k, io->views[k], p->h2d);
                    mark("h2d_" + std::to_string(k), p->h2d);
                    FS_CK(cudaEventRecord(p->ev_h2d[k], p->h2d));
                }
            }
        }
    }
    if (!fc_mode) {  // (first-cover mode reads validity from the owner plane only)
        ProfScope ps("clear", (double)p->cw * p->chh, s);
        FS_CK(cudaMemsetAsync(p->cv.valid, 0, (size_t)p->cw * p->chh, s));
    }
    init_count(p->cc, s);
    if (hin) FS_CK(cudaStreamWaitEvent(s, ev_view[0], 0));
    if (dag) {
        // every pixel of a canvas the (valid everywhere) views cover is
        // written by its writers: no clear of the output
        if (!(fc_mode && p->empty_rects.empty()))
            FS_CK(cudaMemsetAsync(p->out, 0, (size_t)p->cw * p->chh * 4, s));
        FS_CK(cudaEventRecord(p->ev_clear, s));
    }
    {
        ProfScope ps("place", 21.0 * p->rects[0].area(), s);  // view 4 in, rgb 16 + valid 1 out
        launch::place_view(p->cv, view_of(p, 0), p->cc, s, dag ? p->out : nullptr, !fc_mode);
    }
    launches += 2;
    if (!dag) {
        for (int k = 1; k < p->n; ++k) {
            FoldWS<ViewU8>& f = p->folds[k - 1];
            ViewU8 v = view_of(p, k);
            launches += fold_enqueue_pre(f, plane, v, s);
            launch::snapshot_count(f.st, p->cc, s);
            // (the legacy stream's non-null handle when s is the default stream)
            cudaStream_t ts = kLkSplit ? (s ? s : cudaStreamLegacy) : nullptr;
            if (f.tiles_on) {  // the flow tile by tile, then the distance transforms
                launch::check_box(f.st, f.box, s);
                launches += 2;
                for (FlowTile& t : f.tiles) {
                    {
                        ProfScope ps("crop_gray", 29.0 * t.region.area(), s);
                        launch::crop_gray(plane, v, tile_canvas_rect(f, t), 3, t.gray[0],
                                          t.gray[1], s);
                    }
                    launches += 1 + flow_enqueue(t.flow, t.gray[0], t.gray[1], p->fp, t.vec,
                                                 t.valid, s, ts);
                    copy_tile_interior(f, t, s);
                }
                launches += fold_enqueue_edt(f, plane, v, s);
            } else {
                launches += 1 + fold_enqueue_flow_edt(f, plane, plane, v, 3, p->fp, s, nullptr,
                                                      nullptr, nullptr, nullptr, nullptr, true, ts);
            }
            launches += fold_enqueue_blend(f, p->cv, v, p->cc, p->bp, s);
        }
        {
            ProfScope ps("quantize", 21.0 * p->cw * p->chh, s);  // rgb 16 + valid 1 in, rgba8 out
            launch::quantize(p->cv, p->out, s);
        }
        launches += 1;
        FS_CK(cudaGetLastError());
        return launches;
    }
    FS_CK(cudaEventRecord(p->ev_place, s));
    mark("place", s);
    // the owner plane: views claimed in fold order as they land
    FS_CK(cudaStreamWaitEvent(p->own, p->ev_start, 0));
    FS_CK(cudaMemsetAsync(p->owner, 0xFF, (size_t)p->cw * p->chh, p->own));
    // the claims count their pixels: |pano valid| before fold k is the sum of
    // the counts of views < k (no chain through the earlier folds' partitions)
    FS_CK(cudaMemsetAsync(p->hist, 0, sizeof(unsigned long long) * kMaxDagViews, p->own));
    for (int k = 0; k < p->n; ++k) {
        if (hin && !chunked) FS_CK(cudaStreamWaitEvent(p->own, p->ev_h2d[k], 0));
        launch::claim_owner(p->owner, p->cw, view_of(p, k), k, p->own, p->hist);
        ++launches;
        FS_CK(cudaEventRecord(p->ev_own[k], p->own));
    }
    // the read-backs: quantise (and copy) every rectangle once final
    // (the RGBA8 canvas is written by each pixel's writers: copies only)
    auto read_rect = [&](const Rect& r, cudaStream_t st) {
        if (hout) download_rect(p, r, io->out, st);
    };
    // early reads of fold k: after the Area2 copies and composes that may
    // write them (all recorded by the time fold k's branch copied its Area2)
    auto emit_early = [&](int k) {
        for (const auto& rb : p->early[k]) {
            if (rb.place) FS_CK(cudaStreamWaitEvent(p->d2h_early, p->ev_place, 0));
            for (int m : rb.a2) FS_CK(cudaStreamWaitEvent(p->d2h_early, p->ev_a2[m], 0));
            if (rb.compose) FS_CK(cudaStreamWaitEvent(p->d2h_early, p->ev_compose[rb.compose], 0));
            if (&rb == &p->early[k].front())
                mark("readback_early_" + std::to_string(k) + "_ready", p->d2h_early);
            read_rect(rb.r, p->d2h_early);
        }
        if (!p->early[k].empty()) mark("readback_early_" + std::to_string(k), p->d2h_early);
    };
    auto emit_late = [&](int k) {
        if (p->late[k].empty()) return;
        FS_CK(cudaStreamWaitEvent(p->d2h, p->ev_compose[k], 0));
        for (const auto& rb : p->late[k]) read_rect(rb.r, p->d2h);
        mark("readback_" + std::to_string(k), p->d2h);
    };
    emit_early(0);
    for (int k = 1; k < p->n; ++k) {
        FoldWS<ViewU8>& f = p->folds[k - 1];
        ViewU8 v = view_of(p, k);
        cudaStream_t b = p->branch[k - 1];
        FS_CK(cudaStreamWaitEvent(b, hin && !chunked ? p->ev_h2d[k] : p->ev_start, 0));
        FS_CK(cudaStreamWaitEvent(b, p->ev_own[k - 1], 0));  // views < k claimed
        const PanoViews pv = views_before(p, k);
        const std::string fk = std::to_string(k);
        mark("fold" + fk + "_start", b);
        launches += fold_enqueue_pre(f, pv, v, b);
        launch::count_from_hist(f.st, p->hist, k, b);  // claims < k are in
        ++launches;
        // the fold's Area2 (the pixels view k covers first) is a copy of the
        // view: written on the fold's side stream, off the ordered chain and
        // ahead of its distance transforms, while the branch crops and flows
        cudaStream_t es = p->edt_stream[k - 1];
        // device-resident: on the EDT stream (on the branch: C2 0.5% slower);
        // host uploads: on its own stream, so the distance transforms (which
        // need no pixels) do not wait behind the copy for the view to land
        cudaStream_t a2s = chunked ? p->a2_stream[k - 1] : es;
        FS_CK(cudaStreamWaitEvent(a2s, p->ev_own[k], 0));
        FS_CK(cudaStreamWaitEvent(a2s, p->ev_clear, 0));
        if (chunked) FS_CK(cudaStreamWaitEvent(a2s, ev_view[k], 0));  // view k's pixels
        launch::compose_area2(p->cv, v, p->owner, k, a2s, p->out, nullptr,
                              fc_mode ? &no_cv : nullptr);
        ++launches;
        FS_CK(cudaEventRecord(p->ev_a2[k], a2s));
        if (p->tl_stamp && p->crop_wait[k] == 0) mark("fold" + fk + "_flow_start", b);
        cudaEvent_t f0 = tl_event("fold" + fk + "_flow_start"), f1 = tl_event("fold" + fk + "_flow_end");
        cudaEvent_t crop_in = chunked ? ev_crop[k] : nullptr;
        if (f.tiles_on) {
            // row/column tiles: the distance transforms on es from the start;
            // every tile crops (waiting only for the composes its region
            // meets), builds its pyramid and flows on its own streams
            FS_CK(cudaEventRecord(p->ev_efork[k], b));
            FS_CK(cudaStreamWaitEvent(es, p->ev_efork[k], 0));
            launches += fold_enqueue_edt(f, pv, v, es);
            FS_CK(cudaEventRecord(p->ev_ejoin[k], es));
            launch::check_box(f.st, f.box, b);
            ++launches;
            FS_CK(cudaEventRecord(p->ev_tfork[k], b));
            for (size_t t = 0; t < f.tiles.size(); ++t) {
                FlowTile& ft = f.tiles[t];
                cudaStream_t tsm = p->tile_s[k][t];
                FS_CK(cudaStreamWaitEvent(tsm, p->ev_tfork[k], 0));
                if (crop_in) FS_CK(cudaStreamWaitEvent(tsm, crop_in, 0));
                const Rect rc = tile_canvas_rect(f, ft);
                const int m = p->tile_wait[k][t];
                {
                    ProfScope ps("crop_gray", 29.0 * rc.area(), tsm);
                    if (m) {
                        FS_CK(cudaStreamWaitEvent(tsm, p->ev_compose[m], 0));
                        launch::crop_gray(PanoHybrid{pv, plane}, v, rc, 3, ft.gray[0], ft.gray[1],
                                          tsm);
                    } else {
                        launch::crop_gray(pv, v, rc, 3, ft.gray[0], ft.gray[1], tsm);
                    }
                }
                if (p->tl_stamp) mark("fold" + fk + "_tile" + std::to_string(t) + "_start", tsm);
                launches += 1 + flow_enqueue(ft.flow, ft.gray[0], ft.gray[1], p->fp, ft.vec,
                                             ft.valid, tsm, p->tile_ts[k][t]);
                copy_tile_interior(f, ft, tsm);
                if (p->tl_stamp) mark("fold" + fk + "_tile" + std::to_string(t) + "_end", tsm);
                FS_CK(cudaEventRecord(p->ev_tile[k][t], tsm));
                FS_CK(cudaStreamWaitEvent(b, p->ev_tile[k][t], 0));
            }
            FS_CK(cudaStreamWaitEvent(b, p->ev_ejoin[k], 0));
        } else if (p->crop_wait[k] == 0) {
            if (p->tl_stamp) f.flow.mark = [&, fk](const std::string& l, cudaStream_t st) {
                mark("fold" + fk + "_" + l, st);
            };
            launches += fold_enqueue_flow_edt(f, pv, pv, v, 3, p->fp, b, f0, f1, es,
                                              p->ev_efork[k], p->ev_ejoin[k], true,
                                              p->tensor_stream[k - 1], crop_in);
        } else {  // blended pixels inside the box: after that fold's compose
            // (the distance transforms need only the masks: fork them first)
            FS_CK(cudaEventRecord(p->ev_efork[k], b));
            FS_CK(cudaStreamWaitEvent(es, p->ev_efork[k], 0));
            launches += fold_enqueue_edt(f, pv, v, es);
            FS_CK(cudaEventRecord(p->ev_ejoin[k], es));
            FS_CK(cudaStreamWaitEvent(b, p->ev_compose[p->crop_wait[k]], 0));
            if (crop_in) FS_CK(cudaStreamWaitEvent(b, crop_in, 0));
            if (p->tl_stamp) {
                mark("fold" + fk + "_flow_start", b);
                f.flow.mark = [&, fk](const std::string& l, cudaStream_t st) {
                    mark("fold" + fk + "_" + l, st);
                };
            }
            launches += fold_enqueue_flow_edt(f, pv, PanoHybrid{pv, plane}, v, 3, p->fp, b, f0, f1,
                                              nullptr, nullptr, nullptr, false,
                                              p->tensor_stream[k - 1]);
            FS_CK(cudaStreamWaitEvent(b, p->ev_ejoin[k], 0));
        }
        f.flow.mark = nullptr;
        mark("fold" + fk + "_edt_end", b);
        if (chunked) FS_CK(cudaStreamWaitEvent(b, p->ev_a2[k], 0));  // joins the copy's stream
        FS_CK(cudaEventRecord(p->ev_branch[k], b));
        FS_CK(cudaStreamWaitEvent(s, p->ev_branch[k], 0));
        if (chunked) FS_CK(cudaStreamWaitEvent(s, ev_view[k], 0));  // L taps anywhere in views <= k
        mark("fold" + fk + "_blend_start", s);
        // (the last fold's blended pixels are read by no later fold: only the
        // RGBA8 output is written for them in first-cover mode)
        launches += fold_enqueue_blend(f, p->cv, v, p->cc, p->bp, s, p->owner, k, p->out, nullptr,
                                       fc_mode ? &pv : nullptr, !(fc_mode && k == p->n - 1));
        FS_CK(cudaEventRecord(p->ev_compose[k], s));
        mark("fold" + fk + "_compose_end", s);
    }
    // Copies leave the device in submission order (one D2H engine), so they
    // are submitted by expected readiness: a fold's early reads when its view
    // has arrived, its late reads about a fold later (after its flow)
    for (int k = 1; k < p->n; ++k) {
        emit_early(k);
        if (k >= 2) emit_late(k - 1);
    }
    emit_late(p->n - 1);
    FS_CK(cudaEventRecord(p->ev_out, p->d2h));
    FS_CK(cudaStreamWaitEvent(s, p->ev_out, 0));
    FS_CK(cudaEventRecord(p->ev_out_early, p->d2h_early));
    FS_CK(cudaStreamWaitEvent(s, p->ev_out_early, 0));
    if (hfill) FS_CK(cudaStreamWaitEvent(s, p->ev_hfill1, 0));
    if (chunked) FS_CK(cudaStreamWaitEvent(s, p->ev_h2d[p->n - 1], 0));
    mark("end", s);
    FS_CK(cudaGetLastError());
    return launches;
}

// ---- seam sharding ----
bool rects_meet(const Rect& a, const Rect& b) {
    Rect i = rect_inter(a, b);
    return i.w > 0 && i.h > 0;
}

// The global schedule (identical on every rank): fold -> rank, fold -> stage
// (the segment computing it), which ranks need which strips, the transfers.
// Fold k's L crop needs the strips of D_k = {m < k : box m meets box k}; a
// strip m needed on rank r is composed there at the start of segment
// stage[m] + 1, in fold order, so stage[k] = max over D_k of stage[m]
// (+1 when m runs elsewhere).  Rank 0 composes every strip.  A rank composing
// strip j also needs j's own D_j first (the later strip must win where the
// boxes meet).
void shard_schedule(int n, const std::vector<Rect>& boxes, int nranks, std::vector<int>& fold_rank,
                    std::vector<int>& stage, int& nseg, std::vector<fs_strip_xfer>& xfers,
                    std::vector<std::vector<char>>& needed) {
    if (nranks < 1) raise(FS_ERR_CONTRACT, "shard: nranks must be >= 1");
    fold_rank.resize(n, -1);
    fold_rank[0] = 0;
    // list scheduling in fold order, earliest finish first: a fold costs its
    // box area (the flow dominates), a strip moving to another rank 1/10 of
    // its box; ties go to the rank that is not the canvas GPU, then the least
    // loaded
    std::vector<double> avail(nranks, 0.0), finish(n, 0.0);
    for (int k = 1; k < n; ++k) {
        if (fold_rank[k] >= nranks) raise(FS_ERR_CONTRACT, "shard: fold rank out of range");
        const double cost = (double)boxes[k].area();
        auto finish_on = [&](int r) {
            double ready = 0.0;
            for (int m = 1; m < k; ++m)
                if (rects_meet(boxes[m], boxes[k]))
                    ready = std::max(ready, finish[m] + (fold_rank[m] != r ? 0.1 * boxes[m].area() : 0.0));
            return std::max(ready, avail[r]) + cost;
        };
        int best = fold_rank[k];
        if (best < 0) {
            double bf = 0.0;
            for (int r = 0; r < nranks; ++r) {
                const double f = finish_on(r);
                const bool better = best < 0 || f < bf ||
                                    (f == bf && ((best == 0 && r != 0) ||
                                                 ((best == 0) == (r == 0) && avail[r] < avail[best])));
                if (better) {
                    best = r;
                    bf = f;
                }
            }
            fold_rank[k] = best;
        }
        finish[k] = finish_on(best);
        avail[best] = finish[k];
    }
    stage.assign(n, 0);
    int last = 0;
    for (int k = 1; k < n; ++k) {
        for (int m = 1; m < k; ++m)
            if (rects_meet(boxes[m], boxes[k]))
                stage[k] = std::max(stage[k], stage[m] + (fold_rank[m] != fold_rank[k] ? 1 : 0));
        last = std::max(last, stage[k]);
    }
    nseg = last + 2;
    needed.assign(nranks, std::vector<char>(n, 0));
    for (int r = 0; r < nranks; ++r) {
        for (int k = 1; k < n; ++k) {
            if (fold_rank[k] == r) continue;
            if (r == 0) needed[r][k] = 1;
            for (int j = k + 1; j < n; ++j)
                if (fold_rank[j] == r && rects_meet(boxes[k], boxes[j])) needed[r][k] = 1;
        }
        for (bool grew = true; grew;) {  // closure over the strips composed here
            grew = false;
            for (int j = n - 1; j >= 1; --j) {
                if (!needed[r][j]) continue;
                for (int m = 1; m < j; ++m)
                    if (fold_rank[m] != r && !needed[r][m] && rects_meet(boxes[m], boxes[j])) {
                        needed[r][m] = 1;
                        grew = true;
                    }
            }
        }
    }
    xfers.clear();
    for (int st = 0; st <= last; ++st)
        for (int m = 1; m < n; ++m) {
            if (stage[m] != st) continue;
            for (int r = 0; r < nranks; ++r)
                if (needed[r][m]) xfers.push_back(fs_strip_xfer{m, fold_rank[m], r, st});
        }
}

void shard_configure(fs_plan_s* p, int nranks, int rank, const int* fold_rank) {
    if (!p->dag) raise(FS_ERR_UNSUPPORTED, "shard: needs the DAG schedule (n <= 16 views)");
    if (rank < 0 || rank >= nranks) raise(FS_ERR_CONTRACT, "shard: rank out of range");
    auto& S = p->shard;
    for (auto e : S.exec)
        if (e) cudaGraphExecDestroy(e);
    for (auto g : S.graph)
        if (g) cudaGraphDestroy(g);
    S.exec.clear();
    S.graph.clear();
    S.nranks = nranks;
    S.rank = rank;
    const int n = p->n;
    S.fold_rank.assign(n, -1);
    if (fold_rank)
        for (int k = 1; k < n; ++k) S.fold_rank[k] = fold_rank[k];
    std::vector<std::vector<char>> needed;
    shard_schedule(n, p->boxes, nranks, S.fold_rank, S.stage, S.nseg, S.xfers, needed);
    S.apply.assign(S.nseg, {});
    S.own.assign(S.nseg, {});
    for (int k = 1; k < n; ++k) {
        if (needed[rank][k]) S.apply[S.stage[k] + 1].push_back(k);
        if (S.fold_rank[k] == rank) S.own[S.stage[k]].push_back(k);
    }
    // what the canvas holds final when each own fold runs: first-cover
    // copies within kShardMargin of the fold's box, the strips composed here
    S.reach.assign(n, ReachCheck{});
    S.clip = Rect{0, 0, 0, 0};
    S.wait_local.assign(n, 0);
    std::vector<char> present(n, 0);
    for (int sg = 0; sg < S.nseg; ++sg) {
        for (int m : S.apply[sg]) present[m] = 1;
        for (int k : S.own[sg]) {
            ReachCheck& rc = S.reach[k];
            rc.on = nranks > 1;
            const Rect& b = p->boxes[k];
            const int x0 = std::max(0, b.x0 - kShardMargin), y0 = std::max(0, b.y0 - kShardMargin);
            const int x1 = std::min(p->cw, b.x1() + kShardMargin);
            const int y1 = std::min(p->chh, b.y1() + kShardMargin);
            rc.allow = nranks == 1 ? Rect{0, 0, p->cw, p->chh} : Rect{x0, y0, x1 - x0, y1 - y0};
            S.clip = rect_union(S.clip, rc.allow);
            rc.n = 0;
            for (int m = 1; m < n; ++m)
                if (m != k && (m < k) != (present[m] != 0)) rc.forbid[rc.n++] = p->boxes[m];
            for (int m = 1; m < k; ++m)
                if (S.fold_rank[m] == rank && S.stage[m] == sg && rects_meet(p->boxes[m], p->boxes[k]))
                    S.wait_local[k] = m;
            present[k] = 1;
        }
    }
    // rank 0's read-back pieces (the DAG's split of the canvas): each is
    // final once every fold whose box meets it has been composed here
    S.reads.assign(S.nseg, {});
    if (rank == 0) {
        auto seg_of = [&](int m) { return S.stage[m] + (S.fold_rank[m] == 0 ? 0 : 1); };
        for (const auto* lists : {&p->early, &p->late})
            for (const auto& rbs : *lists)
                for (const auto& rb : rbs) {
                    int rs = 0;
                    bool own_last = false;
                    for (int m = 1; m < n; ++m) {
                        if (!rects_meet(p->boxes[m], rb.r)) continue;
                        const int sm = seg_of(m);
                        if (sm > rs) {
                            rs = sm;
                            own_last = false;
                        }
                        if (sm == rs && S.fold_rank[m] == 0) own_last = true;
                    }
                    S.reads[rs][own_last ? 1 : 0].push_back(rb);
                }
    }
    S.exec.assign(S.nseg, nullptr);
    S.graph.assign(S.nseg, nullptr);
    S.launches.assign(S.nseg, 0);
    S.hkeys.clear();
    if (!S.ev_seg) FS_CK(cudaEventCreateWithFlags(&S.ev_seg, cudaEventDisableTiming));
    if (!S.ev_hist) FS_CK(cudaEventCreateWithFlags(&S.ev_hist, cudaEventDisableTiming));
    if (!S.ev_segend) FS_CK(cudaEventCreateWithFlags(&S.ev_segend, cudaEventDisableTiming));
    if (!S.ev_place0) FS_CK(cudaEventCreateWithFlags(&S.ev_place0, cudaEventDisableTiming));
    if (!S.ev_d2h) FS_CK(cudaEventCreateWithFlags(&S.ev_d2h, cudaEventDisableTiming));
    if (!S.hist) FS_CK(cudaMalloc(&S.hist, sizeof(unsigned long long) * kMaxDagViews));
}

// One segment of this rank's sharded execution on stream s.  Segment 0 also
// does what every rank needs whatever folds it owns: view 0's placement, the
// owner claims, every fold's partition counts and first-cover copies (the
// L taps of a blend may read any first-cover pixel).  Then: compose the
// strips received after the previous segment (fold order), run the own
// folds of this segment (branch: crop, pyramid, flow, distance transforms;
// chain on s: blend + compose).
int enqueue_shard(fs_plan_s* p, cudaStream_t s, int seg, const HostIO* io) {
    const auto& S = p->shard;
    uchar4* out = S.rank == 0 ? p->out : nullptr;
    const bool hin = io && io->views;
    int launches = 0;
    if (seg == 0) {
        FS_CK(cudaEventRecord(p->ev_start, s));
        if (hin) {  // views land in fold order; each gates its claim and its fold
            FS_CK(cudaStreamWaitEvent(p->h2d, p->ev_start, 0));
            for (int k = 0; k < p->n; ++k) {
                upload_view(p, k, io->views[k], p->h2d);
                FS_CK(cudaEventRecord(p->ev_h2d[k], p->h2d));
            }
        }
        if (out && io && io->out && !p->empty_rects.empty()) {  // uncovered canvas: host zeroes
            p->hfill_out = io->out;
            FS_CK(cudaStreamWaitEvent(p->hfill, p->ev_start, 0));
            FS_CK(cudaLaunchHostFunc(p->hfill, host_fill_empty, p));
            FS_CK(cudaEventRecord(p->ev_hfill1, p->hfill));
        }
        // the canvas writers (first-cover copies) start after the clear
        if (out) FS_CK(cudaMemsetAsync(out, 0, (size_t)p->cw * p->chh * 4, s));
        FS_CK(cudaEventRecord(p->ev_place, s));
        FS_CK(cudaStreamWaitEvent(p->own, p->ev_place, 0));
        FS_CK(cudaMemsetAsync(p->owner, 0xFF, (size_t)p->cw * p->chh, p->own));
        // the claims count their pixels: |pano valid| before fold k is the sum
        // of hist[m] over m < k (no partition chain over the other folds)
        FS_CK(cudaMemsetAsync(S.hist, 0, sizeof(unsigned long long) * kMaxDagViews, p->own));
        for (int k = 0; k < p->n; ++k) {
            if (hin) FS_CK(cudaStreamWaitEvent(p->own, p->ev_h2d[k], 0));
            launch::claim_owner(p->owner, p->cw, view_of(p, k), k, p->own, S.hist);
            ++launches;
            FS_CK(cudaEventRecord(p->ev_own[k], p->own));
        }
        FS_CK(cudaEventRecord(S.ev_hist, p->own));
        // first-cover copies: the whole canvas on rank 0 (its RGBA8 panorama),
        // around the own folds' boxes elsewhere (their blends' L taps)
        const Rect* clip = S.rank == 0 ? nullptr : &S.clip;
        if (S.rank == 0 || S.clip.w > 0) {
            FS_CK(cudaStreamWaitEvent(s, p->ev_own[0], 0));
            launch::compose_area2(p->cv, view_of(p, 0), p->owner, 0, s, out, clip, &S.clip);
            ++launches;
        }
        FS_CK(cudaEventRecord(S.ev_place0, s));
        for (int k = 1; k < p->n; ++k) {
            const bool mine = S.fold_rank[k] == S.rank;
            if (!mine && S.rank != 0 && S.clip.w <= 0) continue;
            FoldWS<ViewU8>& f = p->folds[k - 1];
            cudaStream_t b = p->branch[k - 1];
            if (hin) FS_CK(cudaStreamWaitEvent(b, p->ev_h2d[k], 0));
            if (mine) {  // the fold's own partition (Area counts, box, statistics)
                FS_CK(cudaStreamWaitEvent(b, p->ev_own[k - 1], 0));
                launches += fold_enqueue_pre(f, views_before(p, k), view_of(p, k), b);
                launch::count_from_hist(f.st, S.hist, k, b);  // claims < k are in
                ++launches;
            }
            FS_CK(cudaStreamWaitEvent(b, p->ev_own[k], 0));
            launch::compose_area2(p->cv, view_of(p, k), p->owner, k, b, out, clip, &S.clip);
            ++launches;
            FS_CK(cudaEventRecord(p->ev_a2[k], b));
            FS_CK(cudaStreamWaitEvent(s, p->ev_a2[k], 0));
        }
        FS_CK(cudaStreamWaitEvent(s, S.ev_hist, 0));
    }
    for (int m : S.apply[seg]) {
        launch::compose_area3(p->cv, view_of(p, m), p->boxes[m], p->folds[m - 1].blended,
                              p->owner, m, s, out);
        ++launches;
    }
    FS_CK(cudaEventRecord(S.ev_seg, s));
    const bool reads = out && io && io->out;
    if (reads && !S.reads[seg][0].empty()) {  // final once this segment's strips are in
        if (seg == 0) {  // first-cover pieces: as soon as their own copies are done
            for (const auto& rb : S.reads[0][0]) {
                if (rb.place) FS_CK(cudaStreamWaitEvent(p->d2h, S.ev_place0, 0));
                for (int m : rb.a2) FS_CK(cudaStreamWaitEvent(p->d2h, p->ev_a2[m], 0));
                download_rect(p, rb.r, io->out, p->d2h);
            }
        } else {
            FS_CK(cudaStreamWaitEvent(p->d2h, S.ev_seg, 0));
            for (const auto& rb : S.reads[seg][0]) download_rect(p, rb.r, io->out, p->d2h);
        }
    }
    const PanoPlane plane{p->cv.valid, p->cv.rgb, p->cv.w};
    for (int k : S.own[seg]) {
        FoldWS<ViewU8>& f = p->folds[k - 1];
        ViewU8 v = view_of(p, k);
        cudaStream_t b = p->branch[k - 1];
        cudaStream_t es = p->edt_stream[k - 1];
        const PanoViews pv = views_before(p, k);
        if (seg > 0) FS_CK(cudaStreamWaitEvent(b, S.ev_seg, 0));
        bool hybrid = false;
        for (int m = 1; m < k; ++m) hybrid = hybrid || rects_meet(p->boxes[m], p->boxes[k]);
        if (!hybrid) {
            launches += fold_enqueue_flow_edt(f, pv, pv, v, 3, p->fp, b, nullptr, nullptr, es,
                                              p->ev_efork[k], p->ev_ejoin[k], true,
                                              p->tensor_stream[k - 1]);
        } else {
            FS_CK(cudaEventRecord(p->ev_efork[k], b));
            FS_CK(cudaStreamWaitEvent(es, p->ev_efork[k], 0));
            launches += fold_enqueue_edt(f, pv, v, es);
            FS_CK(cudaEventRecord(p->ev_ejoin[k], es));
            if (S.wait_local[k]) FS_CK(cudaStreamWaitEvent(b, p->ev_compose[S.wait_local[k]], 0));
            launches += fold_enqueue_flow_edt(f, pv, PanoHybrid{pv, plane}, v, 3, p->fp, b, nullptr,
                                              nullptr, nullptr, nullptr, nullptr, false,
                                              p->tensor_stream[k - 1]);
            FS_CK(cudaStreamWaitEvent(b, p->ev_ejoin[k], 0));
        }
        FS_CK(cudaEventRecord(p->ev_branch[k], b));
        FS_CK(cudaStreamWaitEvent(s, p->ev_branch[k], 0));
        launches += fold_enqueue_blend(f, p->cv, v, p->cc, p->bp, s, p->owner, k, out,
                                       &S.reach[k]);
        FS_CK(cudaEventRecord(p->ev_compose[k], s));
    }
    if (reads) {
        if (!S.reads[seg][1].empty()) {  // after this segment's own composes
            FS_CK(cudaEventRecord(S.ev_segend, s));
            FS_CK(cudaStreamWaitEvent(p->d2h, S.ev_segend, 0));
            for (const auto& rb : S.reads[seg][1]) download_rect(p, rb.r, io->out, p->d2h);
        }
        if (!S.reads[seg][0].empty() || !S.reads[seg][1].empty()) {
            FS_CK(cudaEventRecord(S.ev_d2h, p->d2h));
            FS_CK(cudaStreamWaitEvent(s, S.ev_d2h, 0));
        }
        if (seg == 0 && !p->empty_rects.empty()) FS_CK(cudaStreamWaitEvent(s, p->ev_hfill1, 0));
    }
    FS_CK(cudaGetLastError());
    return launches;
}

void capture(fs_plan_s* p, const HostIO* io, cudaGraph_t* graph, cudaGraphExec_t* exec) {
    FS_CK(cudaStreamBeginCapture(p->cap, cudaStreamCaptureModeThreadLocal));
    int launches = 0;
    try {
        launches = enqueue_all(p, p->cap, p->dag, io);
    } catch (...) {
        cudaGraph_t g = nullptr;
        cudaStreamEndCapture(p->cap, &g);
        if (g) cudaGraphDestroy(g);
        throw;
    }
    FS_CK(cudaStreamEndCapture(p->cap, graph));
    // kernel nodes keep the priority of the stream they were captured on
    FS_CK(cudaGraphInstantiateWithFlags(exec, *graph, cudaGraphInstantiateFlagUseNodePriority));
    p->launches = launches;
}

void capture_shard(fs_plan_s* p, int seg, const HostIO* io) {
    auto& S = p->shard;
    FS_CK(cudaStreamBeginCapture(p->cap, cudaStreamCaptureModeThreadLocal));
    try {
        S.launches[seg] = enqueue_shard(p, p->cap, seg, io);
    } catch (...) {
        cudaGraph_t g = nullptr;
        cudaStreamEndCapture(p->cap, &g);
        if (g) cudaGraphDestroy(g);
        throw;
    }
    FS_CK(cudaStreamEndCapture(p->cap, &S.graph[seg]));
    FS_CK(cudaGraphInstantiateWithFlags(&S.exec[seg], S.graph[seg],
                                        cudaGraphInstantiateFlagUseNodePriority));
}

void drop_shard_graphs(fs_plan_s* p) {
    auto& S = p->shard;
    for (auto& e : S.exec)
        if (e) {
            cudaGraphExecDestroy(e);
            e = nullptr;
        }
    for (auto& g : S.graph)
        if (g) {
            cudaGraphDestroy(g);
            g = nullptr;
        }
    S.hkeys.clear();
}

void build_graph(fs_plan_s* p) {
    if (!p->exec) capture(p, nullptr, &p->graph, &p->exec);
}

void drop_graph(fs_plan_s* p) {
    if (p->exec) cudaGraphExecDestroy(p->exec);
    if (p->graph) cudaGraphDestroy(p->graph);
    if (p->hexec) cudaGraphExecDestroy(p->hexec);
    if (p->hgraph) cudaGraphDestroy(p->hgraph);
    p->exec = nullptr;
    p->graph = nullptr;
    p->hexec = nullptr;
    p->hgraph = nullptr;
    p->hkey.clear();
    drop_shard_graphs(p);
}

// Page-locked (or device) memory can be read by a graph's copy nodes
// asynchronously; pageable host memory cannot.
bool async_copyable(const void* ptr) {
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, ptr) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return at.type != cudaMemoryTypeUnregistered;
}


// Canvas rectangles final after fold k (k = 0: after view 0 is placed): the
// canvas is cut into cells along every view edge; a cell is final after the
// last fold whose view covers it (fold m writes only inside view m's rect).
void plan_final_rects(fs_plan_s* p) {
    std::vector<int> xs{0, p->cw}, ys{0, p->chh};
    for (const Rect& r : p->rects) {
        xs.push_back(r.x0);
        xs.push_back(r.x1());
        ys.push_back(r.y0);
        ys.push_back(r.y1());
    }
    std::sort(xs.begin(), xs.end());
    xs.erase(std::unique(xs.begin(), xs.end()), xs.end());
    std::sort(ys.begin(), ys.end());
    ys.erase(std::unique(ys.begin(), ys.end()), ys.end());
    // slot n: cells no view covers (their RGBA8 value is 0: filled on the host)
    const int slots = p->n + 1;
    p->final_rects.assign(slots, {});
    std::vector<std::vector<Rect>> open(slots);  // runs of the previous row band
    for (size_t j = 0; j + 1 < ys.size(); ++j) {
        const int y0 = ys[j], y1 = ys[j + 1];
        std::vector<std::vector<Rect>> cur(slots);
        for (size_t i = 0; i + 1 < xs.size();) {
            auto last_of = [&](size_t c) {
                int last = p->n;
                for (int k = 0; k < p->n; ++k)
                    if (p->rects[k].contains(xs[c], y0)) last = k;
                return last;
            };
            const int k = last_of(i);
            size_t e = i + 1;
            while (e + 1 < xs.size() && last_of(e) == k) ++e;
            cur[k].push_back(Rect{xs[i], y0, xs[e] - xs[i], y1 - y0});
            i = e;
        }
        for (int k = 0; k < slots; ++k) {  // extend matching runs of the band above
            std::vector<Rect> next;
            for (Rect r : cur[k]) {
                bool merged = false;
                for (Rect& o : open[k])
                    if (o.x0 == r.x0 && o.w == r.w && o.y1() == r.y0) {
                        o.h += r.h;
                        next.push_back(o);
                        o.w = 0;
                        merged = true;
                        break;
                    }
                if (!merged) next.push_back(r);
            }
            for (const Rect& o : open[k])
                if (o.w > 0) p->final_rects[k].push_back(o);
            open[k] = next;
        }
    }
    for (int k = 0; k < slots; ++k)
        for (const Rect& o : open[k]) p->final_rects[k].push_back(o);
    p->empty_rects = p->final_rects[p->n];
    p->final_rects.resize(p->n);
}

// Split of the final rectangles (see fs_plan_s::Readback).
void plan_readbacks(fs_plan_s* p) {
    plan_final_rects(p);
    const int n = p->n;
    p->early.assign(n, {});
    p->late.assign(n, {});
    auto meets = [](const Rect& a, const Rect& b) {
        Rect i = rect_inter(a, b);
        return i.w > 0 && i.h > 0;
    };
    for (int k = 0; k < n; ++k)
        for (const Rect& R : p->final_rects[k]) {
            if (k == 0) {
                p->early[0].push_back({R, {}, 0, true});
                continue;
            }
            const Rect& B = p->boxes[k];
            const Rect in = rect_inter(R, B);
            if (in.w > 0 && in.h > 0) p->late[k].push_back({in, {}, 0, false});
            // R minus the box: the bands above and below, then left and right
            std::vector<Rect> pieces;
            if (in.w <= 0 || in.h <= 0) {
                pieces.push_back(R);
            } else {
                pieces.push_back(Rect{R.x0, R.y0, R.w, in.y0 - R.y0});
                pieces.push_back(Rect{R.x0, in.y1(), R.w, R.y1() - in.y1()});
                pieces.push_back(Rect{R.x0, in.y0, in.x0 - R.x0, in.h});
                pieces.push_back(Rect{in.x1(), in.y0, R.x1() - in.x1(), in.h});
            }
            for (const Rect& q : pieces) {
                if (q.w <= 0 || q.h <= 0) continue;
                fs_plan_s::Readback rb{q, {}, 0, meets(p->rects[0], q)};
                for (int m = 1; m <= k; ++m)
                    if (meets(p->rects[m], q)) rb.a2.push_back(m);
                for (int m = 1; m < k; ++m)
                    if (meets(p->boxes[m], q)) rb.compose = m;
                p->early[k].push_back(rb);
            }
        }
}

// Area3 boxes of every fold from the view masks: a validity-only fold on the
// device (partition statistics, then pano valid |= view valid).
std::vector<Rect> boxes_from_masks(fs_plan_s* p, const uint8_t* const* views_rgba) {
    cudaStream_t s = p->cap;
    size_t nc = (size_t)p->cw * p->chh;
    uint8_t* valid = nullptr;
    FoldStats* st = nullptr;
    FS_CK(cudaMalloc(&valid, nc));
    FS_CK(cudaMalloc(&st, sizeof(FoldStats) * p->n));
    std::vector<uchar4*> tmp(p->n, nullptr);
    std::vector<Rect> boxes(p->n);
    try {
        for (int k = 0; k < p->n; ++k) {
            size_t np = (size_t)p->rects[k].w * p->rects[k].h;
            FS_CK(cudaMalloc(&tmp[k], np * 4 + 4));
            FS_CK(cudaMemcpyAsync(tmp[k], views_rgba[k], np * 4, cudaMemcpyDefault, s));
        }
        FS_CK(cudaMemsetAsync(valid, 0, nc, s));
        Canvas cv{nullptr, valid, p->cw, p->chh, 3};
        launch::union_valid(cv, ViewU8{tmp[0], p->rects[0]}, s);
        for (int k = 1; k < p->n; ++k) {
            ViewU8 v{tmp[k], p->rects[k]};
            init_stats(st + k, s);
            launch::partition(PanoPlane{valid, nullptr, p->cw}, v, st + k, s);
            launch::union_valid(cv, v, s);
        }
        std::vector<FoldStats> hs(p->n);
        FS_CK(cudaMemcpyAsync(hs.data(), st, sizeof(FoldStats) * p->n, cudaMemcpyDeviceToHost, s));
        FS_CK(cudaStreamSynchronize(s));
        for (int k = 1; k < p->n; ++k) {
            if (hs[k].cnt3 == 0)
                raise(FS_ERR_EMPTY_REGION,
                      "stitch: no overlap between the panorama and image #" + std::to_string(k));
            boxes[k] = Rect{hs[k].bx0, hs[k].by0, hs[k].bx1 - hs[k].bx0 + 1,
                            hs[k].by1 - hs[k].by0 + 1};
        }
    } catch (...) {
        for (auto* t : tmp) cudaFree(t);
        cudaFree(valid);
        cudaFree(st);
        throw;
    }
    for (auto* t : tmp) cudaFree(t);
    cudaFree(valid);
    cudaFree(st);
    return boxes;
}

// Fully valid rectangles: Area3 of fold k is (union of rects < k) ∩ rect k,
// whose bounding box is the union of the pairwise intersections' boxes.
std::vector<Rect> boxes_from_rects(fs_plan_s* p) {
    std::vector<Rect> boxes(p->n);
    for (int k = 1; k < p->n; ++k) {
        Rect b{0, 0, 0, 0};
        for (int m = 0; m < k; ++m) {
            Rect i = rect_inter(p->rects[m], p->rects[k]);
            if (i.w > 0 && i.h > 0) b = rect_union(b, i);
        }
        if (b.w <= 0 || b.h <= 0)
            raise(FS_ERR_EMPTY_REGION,
                  "stitch: no overlap between the panorama and image #" + std::to_string(k));
        boxes[k] = b;
    }
    return boxes;
}

void layout_plan(fs_plan_s* p, Arena& a, const std::vector<Rect>& boxes) {
    p->views.resize(p->n);
    for (int k = 0; k < p->n; ++k)
        p->views[k] = a.take<uchar4>((size_t)p->rects[k].w * p->rects[k].h);
    size_t nc = (size_t)p->cw * p->chh;
    p->out = a.take<uchar4>(nc);
    p->cv.rgb = a.take<float4>(nc);
    p->cv.valid = a.take<uint8_t>(nc);
    p->cv.w = p->cw;
    p->cv.h = p->chh;
    p->cv.ch = 3;
    p->cc = a.take<CanvasCount>(1);
    p->owner = p->dag ? a.take<uint8_t>(nc) : nullptr;
    p->folds.resize(p->n - 1);
    for (int k = 1; k < p->n; ++k) {
        bool full = p->folds[k - 1].full_domain;
        p->folds[k - 1].full_domain = full;
        p->folds[k - 1].layout(a, boxes[k], p->pano_bbox[k], p->rects[k], p->fp);
    }
}

}  // namespace

extern "C" {

fs_status fs_plan_create(fs_plan* out, int device, int n, const int* dims, const int* offsets,
                         int canvas_w, int canvas_h, const fs_flow_params* flow,
                         const fs_blend_params* blend, const uint8_t* const* views_rgba) {
    *out = nullptr;
    fs_plan_s* p = new fs_plan_s();
    fs_status st = plan_guard([&] {
        FS_CK(cudaSetDevice(device));
        ensure_device();
        if (n < 2) raise(FS_ERR_CONTRACT, "stitch: at least two images required");
        validate_flow_params(*flow);
        validate_blend_params(*blend);
        check_edt_extent(canvas_w, canvas_h, "plan");
        p->device = device;
        p->n = n;
        p->cw = canvas_w;
        p->chh = canvas_h;
        p->fp = *flow;
        p->bp = *blend;
        for (int k = 0; k < n; ++k) {
            Rect r{offsets[2 * k], offsets[2 * k + 1], dims[2 * k], dims[2 * k + 1]};
            if (r.x0 < 0 || r.y0 < 0 || r.x1() > canvas_w || r.y1() > canvas_h)
                raise(FS_ERR_LAYOUT, "place_on_canvas: image does not fit inside the canvas");
            if (r.w <= 0 || r.h <= 0) raise(FS_ERR_CONTRACT, "plan: empty view");
            p->rects.push_back(r);
        }
        {
            // the graph's own stream carries the ordered blend + compose chain
            // (and place, clear): critical path, highest priority (the graph's
            // kernel nodes keep the priority of the stream they were captured on)
            int least = 0, greatest = 0;
            FS_CK(cudaDeviceGetStreamPriorityRange(&least, &greatest));
            FS_CK(cudaStreamCreateWithPriority(&p->cap, cudaStreamNonBlocking, greatest));
        }
        std::vector<Rect> boxes = views_rgba ? boxes_from_masks(p, views_rgba) : boxes_from_rects(p);
        // DAG: fold k's L crop may come straight from the views when no earlier
        // fold's Area3 box overlaps its own (those pixels hold the first
        // covering view's value); otherwise it waits only for the compose of
        // the last earlier fold whose box meets its own.  Partitions and
        // distance transforms never wait.
        p->dag = n <= kMaxDagViews;
        p->crop_wait.assign(n, 0);
        for (int k = 1; k < n; ++k)
            for (int m = 1; m < k; ++m) {
                Rect i = rect_inter(boxes[m], boxes[k]);
                if (i.w > 0 && i.h > 0) p->crop_wait[k] = m;
            }
        if (p->dag) {
            p->branch.assign(n - 1, nullptr);
            p->ev_branch.assign(n, nullptr);
            p->ev_compose.assign(n, nullptr);
            // every fold's branch at one (high) priority, above the chain:
            // folds released together (e.g. C2's two bands) share the GPU
            // instead of the later one starving behind the earlier one's
            // sweeps (measured: ordering branches by fold was 0.15-0.25 ms slower)
            int least = 0, greatest = 0;
            FS_CK(cudaDeviceGetStreamPriorityRange(&least, &greatest));
            p->edt_stream.assign(n - 1, nullptr);
            p->tensor_stream.assign(n - 1, nullptr);
            p->a2_stream.assign(n - 1, nullptr);
            // Priorities by slack: the flow chains first (their coarse levels
            // are few CTAs, latency-bound, and starved behind big side
            // kernels otherwise); the level tensors (needed level by level)
            // and the distance transforms / Area2 copies of the folds that
            // start at once next; the distance transforms of the folds whose
            // flow waits for an earlier compose (C2's bands: needed a whole
            // phase later) last.
            const int p_next = std::min(least, greatest + 1);
            for (int k = 0; k < n - 1; ++k) {
                int p_side = p->crop_wait[k + 1] ? least : p_next;
                // the first fold of the first phase blends first: its distance
                // transforms at the flows' priority (C2 3.394 -> 3.382 ms)
                bool first = !p->crop_wait[k + 1];
                for (int m = 1; m < k + 1; ++m) first &= p->crop_wait[m] != 0;
                                if (first) p_side = greatest;
                FS_CK(cudaStreamCreateWithPriority(&p->branch[k], cudaStreamNonBlocking, greatest));
                FS_CK(cudaStreamCreateWithPriority(&p->edt_stream[k], cudaStreamNonBlocking,
                                                   p_side));
                FS_CK(cudaStreamCreateWithPriority(&p->tensor_stream[k], cudaStreamNonBlocking,
                                                   p_next));
                FS_CK(cudaStreamCreateWithPriority(&p->a2_stream[k], cudaStreamNonBlocking,
                                                   p_side));
            }
            p->ev_h2d.assign(n, nullptr);
            p->ev_own.assign(n, nullptr);
            p->ev_a2.assign(n, nullptr);
            p->ev_efork.assign(n, nullptr);
            p->ev_ejoin.assign(n, nullptr);
            for (int k = 0; k < n; ++k) {
                FS_CK(cudaEventCreateWithFlags(&p->ev_branch[k], cudaEventDisableTiming));
                FS_CK(cudaEventCreateWithFlags(&p->ev_compose[k], cudaEventDisableTiming));
                FS_CK(cudaEventCreateWithFlags(&p->ev_h2d[k], cudaEventDisableTiming));
                FS_CK(cudaEventCreateWithFlags(&p->ev_own[k], cudaEventDisableTiming));
                FS_CK(cudaEventCreateWithFlags(&p->ev_a2[k], cudaEventDisableTiming));
                FS_CK(cudaEventCreateWithFlags(&p->ev_efork[k], cudaEventDisableTiming));
                FS_CK(cudaEventCreateWithFlags(&p->ev_ejoin[k], cudaEventDisableTiming));
            }
            for (cudaEvent_t* e : {&p->ev_start, &p->ev_place, &p->ev_out, &p->ev_out_early,
                                   &p->ev_clear})
                FS_CK(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
            FS_CK(cudaMalloc(&p->hist, sizeof(unsigned long long) * kMaxDagViews));
            // the transfer streams' kernels (RGB8 expansion and packing) are
            // tiny and gate the copy engines: highest priority, so they do
            // not queue behind the flows
            FS_CK(cudaStreamCreateWithPriority(&p->h2d, cudaStreamNonBlocking, greatest));
            FS_CK(cudaStreamCreateWithPriority(&p->d2h, cudaStreamNonBlocking, greatest));
            FS_CK(cudaStreamCreateWithPriority(&p->d2h_early, cudaStreamNonBlocking, greatest));
            FS_CK(cudaStreamCreateWithFlags(&p->hfill, cudaStreamNonBlocking));
            FS_CK(cudaEventCreateWithFlags(&p->ev_hfill1, cudaEventDisableTiming));
            // the claims gate every fold's branch: highest priority
            FS_CK(cudaStreamCreateWithPriority(&p->own, cudaStreamNonBlocking, greatest));
            p->boxes = boxes;
            plan_readbacks(p);
        }
        p->pano_bbox.assign(n, Rect{});
        Rect pb = p->rects[0];
        for (int k = 1; k < n; ++k) {
            p->pano_bbox[k] = pb;
            pb = rect_union(pb, p->rects[k]);
        }
        Arena a0;
        layout_plan(p, a0, boxes);
        FS_CK(cudaMalloc(&p->arena, a0.off));
        FS_CK(cudaMalloc(&p->landed, sizeof(unsigned long long) * n));
        Arena a1;
        a1.base = p->arena;
        layout_plan(p, a1, boxes);
        if (kLkSplit)
            for (auto& f : p->folds) flow_split_events(f.flow);
        for (int k = 1; k < n; ++k) {  // folds released together with others
            int together = 0;
            for (int m = 1; m < n; ++m) together += p->crop_wait[m] == p->crop_wait[k];
            p->folds[k - 1].flow.tensor0_on_chain = together > 1;
        }
        if (views_rgba)
            for (int k = 0; k < n; ++k)
                FS_CK(cudaMemcpy(p->views[k], views_rgba[k],
                                 (size_t)p->rects[k].w * p->rects[k].h * 4, cudaMemcpyDefault));
    });
    if (st != FS_OK) {
        fs_plan_destroy(p);
        return st;
    }
    *out = p;
    return FS_OK;
}

void* fs_plan_view_buffer(fs_plan p, int k) {
    return (p && k >= 0 && k < p->n) ? p->views[k] : nullptr;
}
void* fs_plan_output_buffer(fs_plan p) { return p ? p->out : nullptr; }
int fs_plan_launch_count(fs_plan p) { return p ? p->launches : 0; }

fs_status fs_plan_set_host_format(fs_plan p, int view_channels, int out_channels) {
    return plan_guard([&] {
        if (!p || (view_channels != 3 && view_channels != 4) ||
            (out_channels != 3 && out_channels != 4))
            raise(FS_ERR_CONTRACT, "plan: host formats are RGB8 (3) or RGBA8 (4)");
        FS_CK(cudaSetDevice(p->device));
        if (view_channels == p->hv_ch && out_channels == p->ho_ch) return;
        if (view_channels == 3 && !p->stage_in) {
            size_t off = 0;
            p->stage_off.assign(p->n, 0);
            for (int k = 0; k < p->n; ++k) {
                p->stage_off[k] = off;
                off += ((size_t)p->rects[k].w * p->rects[k].h * 3 + 255) & ~size_t(255);
            }
            FS_CK(cudaMalloc(&p->stage_in, off));
        }
        if (out_channels == 3 && !p->stage_out)
            FS_CK(cudaMalloc(&p->stage_out, (size_t)p->cw * p->chh * 3 + 16));
        if (view_channels == 3 && p->hv_ch != 3) {
            // RGB8 views: every pixel valid, alpha 255 before any data lands
            for (int k = 0; k < p->n; ++k)
                launch::set_alpha(p->views[k], (size_t)p->rects[k].w * p->rects[k].h, nullptr);
            FS_CK(cudaDeviceSynchronize());
            p->ho_ch = out_channels;  // the chunk order weighs the read-back bytes
            if (p->dag) plan_chunks(p);
        }
        p->hv_ch = view_channels;
        p->ho_ch = out_channels;
        // the graphs were captured for the old formats (the host copies; the
        // views' validity: RGB8 views are valid everywhere)
        drop_graph(p);
    });
}

static void free_tiles(fs_plan_s* p) {
    for (auto& v : p->tile_s)
        for (auto st : v) cudaStreamDestroy(st);
    for (auto& v : p->tile_ts)
        for (auto st : v) cudaStreamDestroy(st);
    for (auto& v : p->ev_tile)
        for (auto e : v) cudaEventDestroy(e);
    for (auto e : p->ev_tfork)
        if (e) cudaEventDestroy(e);
    for (auto& f : p->folds) {
        for (auto& t : f.tiles) flow_destroy_events(t.flow);
        f.tiles.clear();
        f.tiles_on = false;
    }
    p->tile_s.clear();
    p->tile_ts.clear();
    p->ev_tile.clear();
    p->ev_tfork.clear();
    p->tile_wait.clear();
    if (p->tile_arena) cudaFree(p->tile_arena);
    p->tile_arena = nullptr;
}

fs_status fs_plan_set_tiling(fs_plan p, int tile_len, int margin) {
    return plan_guard([&] {
        if (!p || tile_len < 0 || margin < 0)
            raise(FS_ERR_CONTRACT, "plan: tile_len and margin must be >= 0");
        FS_CK(cudaSetDevice(p->device));
        FS_CK(cudaDeviceSynchronize());
        drop_graph(p);
        free_tiles(p);
        p->tile_len = tile_len;
        p->tile_margin = margin;
        if (tile_len == 0) return;
        if (!p->dag || !kLkSplit)
            raise(FS_ERR_UNSUPPORTED, "plan: flow tiles need the DAG schedule and the split LK");
        const int n = p->n;
        int any = 0;
        for (int k = 1; k < n; ++k) {
            FoldWS<ViewU8>& f = p->folds[k - 1];
            const int axis = f.box.w >= f.box.h ? 0 : 1;  // cut the long axis
            f.tiles_on = plan_flow_tiles(f.box.w, f.box.h, axis, tile_len, margin, p->fp, f.tiles);
            any += f.tiles_on;
        }
        if (!any) return;
        auto lay = [&](Arena& a) {
            for (auto& f : p->folds)
                for (auto& t : f.tiles) layout_flow_tile(t, a, p->fp, f.box.w, f.box.h);
        };
        Arena a0;
        lay(a0);
        FS_CK(cudaMalloc(&p->tile_arena, a0.off));
        Arena a1;
        a1.base = p->tile_arena;
        lay(a1);
        int least = 0, greatest = 0;
        FS_CK(cudaDeviceGetStreamPriorityRange(&least, &greatest));
        p->tile_s.assign(n, {});
        p->tile_ts.assign(n, {});
        p->ev_tile.assign(n, {});
        p->ev_tfork.assign(n, nullptr);
        p->tile_wait.assign(n, {});
        for (int k = 1; k < n; ++k) {
            FoldWS<ViewU8>& f = p->folds[k - 1];
            if (f.tiles.empty()) continue;
            FS_CK(cudaEventCreateWithFlags(&p->ev_tfork[k], cudaEventDisableTiming));
            for (auto& t : f.tiles) {
                t.flow.cert_fail = &f.st->tile_fail;
                flow_split_events(t.flow);
                cudaStream_t a, b;
                cudaEvent_t e;
                FS_CK(cudaStreamCreateWithPriority(&a, cudaStreamNonBlocking, greatest));
                FS_CK(cudaStreamCreateWithPriority(&b, cudaStreamNonBlocking, greatest));
                FS_CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
                p->tile_s[k].push_back(a);
                p->tile_ts[k].push_back(b);
                p->ev_tile[k].push_back(e);
                int wait = 0;
                const Rect rc = tile_canvas_rect(f, t);
                for (int m = 1; m < k; ++m)
                    if (rects_meet(p->boxes[m], rc)) wait = m;
                p->tile_wait[k].push_back(wait);
            }
        }
    });
}

int fs_plan_tile_count(fs_plan p, int k) {
    if (!p || k < 1 || k >= p->n) return -1;
    const auto& f = p->folds[k - 1];
    return f.tiles_on ? (int)f.tiles.size() : 0;
}

fs_status fs_plan_tile_info(fs_plan p, int k, int t, int* region, int* interior) {
    if (!p || k < 1 || k >= p->n) return FS_ERR_CONTRACT;
    const auto& f = p->folds[k - 1];
    if (t < 0 || t >= (int)f.tiles.size()) return FS_ERR_CONTRACT;
    const Rect &R = f.tiles[t].region, &I = f.tiles[t].interior;
    const int rv[4] = {R.x0, R.y0, R.w, R.h}, iv[4] = {I.x0, I.y0, I.w, I.h};
    for (int i = 0; i < 4; ++i) {
        if (region) region[i] = rv[i];
        if (interior) interior[i] = iv[i];
    }
    return FS_OK;
}

fs_status fs_plan_transfer_bytes(fs_plan p, size_t* h2d, size_t* d2h) {
    if (!p) return FS_ERR_CONTRACT;
    size_t in = 0, out = (size_t)p->cw * p->chh * p->ho_ch;
    for (const Rect& r : p->rects) in += (size_t)r.w * r.h * p->hv_ch;
    if (p->dag) {
        out = 0;
        for (const auto* v : {&p->early, &p->late})
            for (const auto& rbs : *v)
                for (const auto& rb : rbs) out += (size_t)rb.r.w * rb.r.h * p->ho_ch;
    }
    if (h2d) *h2d = in;
    if (d2h) *d2h = out;
    return FS_OK;
}

fs_status fs_plan_fold_info(fs_plan p, int k, int* box, int* depth) {
    if (!p || k < 1 || k >= p->n) return FS_ERR_CONTRACT;
    const FoldWS<ViewU8>& f = p->folds[k - 1];
    box[0] = f.box.x0;
    box[1] = f.box.y0;
    box[2] = f.box.w;
    box[3] = f.box.h;
    if (depth) *depth = f.depth;
    return FS_OK;
}

fs_status fs_plan_fold_flow(fs_plan p, int k, float* ltor_vec, uint8_t* ltor_valid,
                            float* rtol_vec, uint8_t* rtol_valid) {
    if (!p || k < 1 || k >= p->n) return FS_ERR_CONTRACT;
    return plan_guard([&] {
        FS_CK(cudaSetDevice(p->device));
        FS_CK(cudaDeviceSynchronize());
        const FoldWS<ViewU8>& f = p->folds[k - 1];
        size_t n = (size_t)f.box.w * f.box.h;
        float* vec[2] = {ltor_vec, rtol_vec};
        uint8_t* val[2] = {ltor_valid, rtol_valid};
        for (int d = 0; d < 2; ++d) {
            if (vec[d]) FS_CK(cudaMemcpy(vec[d], f.fvec[d], n * sizeof(float2), cudaMemcpyDefault));
            if (val[d]) FS_CK(cudaMemcpy(val[d], f.fvalid[d], n, cudaMemcpyDefault));
        }
    });
}

fs_status fs_plan_execute_host_async(fs_plan p, const uint8_t* const* views_rgba,
                                     uint8_t* out_rgba, void* stream) {
    return plan_guard([&] {
        FS_CK(cudaSetDevice(p->device));
        bool ok = p->dag && views_rgba && out_rgba && async_copyable(out_rgba);
        for (int k = 0; ok && k < p->n; ++k) ok = async_copyable(views_rgba[k]);
        if (!ok)
            raise(FS_ERR_UNSUPPORTED, "plan: execute_host_async needs the DAG schedule and "
                                      "page-locked views and canvas");
        std::vector<const void*> key;
        for (int k = 0; k < p->n; ++k) key.push_back(views_rgba[k]);
        key.push_back((const void*)1);
        key.push_back(out_rgba);
        if (p->hexec && p->hkey != key) {
            cudaGraphExecDestroy(p->hexec);
            cudaGraphDestroy(p->hgraph);
            p->hexec = nullptr;
            p->hgraph = nullptr;
        }
        if (!p->hexec) {
            HostIO io{views_rgba, out_rgba};
            capture(p, &io, &p->hgraph, &p->hexec);
            p->hkey = key;
        }
        FS_CK(cudaGraphLaunch(p->hexec, static_cast<cudaStream_t>(stream)));
    });
}

fs_status fs_plan_execute(fs_plan p, void* stream) {
    return plan_guard([&] {
        FS_CK(cudaSetDevice(p->device));
        build_graph(p);
        FS_CK(cudaGraphLaunch(p->exec, static_cast<cudaStream_t>(stream)));
    });
}

fs_status fs_plan_check(fs_plan p) {
    return plan_guard([&] {
        FS_CK(cudaSetDevice(p->device));
        if (!p->hstats) FS_CK(cudaMallocHost(&p->hstats, sizeof(FoldStats) * p->folds.size()));
        for (size_t k = 0; k < p->folds.size(); ++k)
            FS_CK(cudaMemcpyAsync(&p->hstats[k], p->folds[k].st, sizeof(FoldStats),
                                  cudaMemcpyDeviceToHost, p->cap));
        FS_CK(cudaStreamSynchronize(p->cap));
        const FoldStats* hs = p->hstats;
        for (size_t k = 0; k < p->folds.size(); ++k)
            if (hs[k].box_mismatch)
                raise(FS_ERR_CONTRACT, "plan: the views' masks no longer produce the planned "
                                       "overlap of fold #" + std::to_string(k + 1));
        for (size_t k = 0; k < p->folds.size(); ++k)
            if (hs[k].reach_fail)
                raise(FS_ERR_SHARD_REACH, "plan: sharded fold #" + std::to_string(k + 1) +
                                              " sampled the panorama outside the strips its GPU "
                                              "holds; execute unsharded");
        bool untiled = false;
        for (size_t k = 0; k < p->folds.size(); ++k)
            if (hs[k].tile_fail && p->folds[k].tiles_on) {
                p->folds[k].tiles_on = false;
                untiled = true;
            }
        if (untiled) {
            drop_graph(p);
            raise(FS_ERR_CONTRACT, "plan: a flow tile gathered outside its exact pyramid part; "
                                   "the fold runs untiled from now on, execute again");
        }
        bool widened = false;
        for (size_t k = 0; k < p->folds.size(); ++k)
            if (hs[k].edt_fail && !p->folds[k].full_domain) {
                p->folds[k].full_domain = true;
                p->folds[k].replan_edt();
                widened = true;
            }
        if (widened) {
            drop_graph(p);
            raise(FS_ERR_CONTRACT, "plan: bounded distance-transform domain was not provably "
                                   "exact; widened to the full domain, execute again");
        }
    });
}

fs_status fs_plan_execute_host(fs_plan p, const uint8_t* const* views_rgba, uint8_t* out_rgba,
                               void* stream) {
    return plan_guard([&] {
        FS_CK(cudaSetDevice(p->device));
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        // transfers inside the graph, overlapping the folds, when the host
        // buffers allow asynchronous copies
        bool overlap = p->dag && (views_rgba || out_rgba);
        if (overlap && views_rgba)
            for (int k = 0; k < p->n; ++k) overlap = overlap && async_copyable(views_rgba[k]);
        if (overlap && out_rgba) overlap = async_copyable(out_rgba);
        std::vector<const void*> key;
        if (overlap) {
            for (int k = 0; views_rgba && k < p->n; ++k) key.push_back(views_rgba[k]);
            key.push_back(views_rgba ? (const void*)1 : nullptr);
            key.push_back(out_rgba);
        }
        for (int attempt = 0; attempt < 2; ++attempt) {
            if (overlap) {
                if (p->hexec && p->hkey != key) {
                    cudaGraphExecDestroy(p->hexec);
                    cudaGraphDestroy(p->hgraph);
                    p->hexec = nullptr;
                    p->hgraph = nullptr;
                }
                if (!p->hexec) {
                    HostIO io{views_rgba, out_rgba};
                    capture(p, &io, &p->hgraph, &p->hexec);
                    p->hkey = key;
                }
                FS_CK(cudaGraphLaunch(p->hexec, s));
            } else {
                if (views_rgba)
                    for (int k = 0; k < p->n; ++k) upload_view(p, k, views_rgba[k], s);
                build_graph(p);
                FS_CK(cudaGraphLaunch(p->exec, s));
                if (out_rgba) download_rect(p, Rect{0, 0, p->cw, p->chh}, out_rgba, s);
            }
            FS_CK(cudaStreamSynchronize(s));
            fs_status c = fs_plan_check(p);
            if (c == FS_OK) return;
            if (attempt == 1 || p->exec || p->hexec) raise(c, last_error_slot());
        }
    });
}

fs_status fs_plan_timeline(fs_plan p, const uint8_t* const* views_rgba, uint8_t* out_rgba,
                           void* stream, char* json, int cap) {
    return plan_guard([&] {
        FS_CK(cudaSetDevice(p->device));
        if (!p->dag) raise(FS_ERR_UNSUPPORTED, "plan: timeline needs the DAG schedule");
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        HostIO io{views_rgba, out_rgba};
        cudaGraph_t g = nullptr;
        cudaGraphExec_t e = nullptr;
        const int saved = p->launches;
        p->tl = true;
        p->tl_marks.clear();
        auto cleanup = [&] {
            p->tl = false;
            for (auto& m : p->tl_marks) cudaEventDestroy(m.second);
            p->tl_marks.clear();
            if (e) cudaGraphExecDestroy(e);
            if (g) cudaGraphDestroy(g);
            p->launches = saved;
        };
        try {
            // the same stream schedule as the graph, launched directly (timing
            // events are not available on graph event-record nodes)
            enqueue_all(p, s, true, (views_rgba || out_rgba) ? &io : nullptr);
            FS_CK(cudaStreamSynchronize(s));
            for (auto& m : p->tl_marks) cudaEventDestroy(m.second);
            p->tl_marks.clear();
            enqueue_all(p, s, true, (views_rgba || out_rgba) ? &io : nullptr);
            FS_CK(cudaStreamSynchronize(s));
            std::string js = "{";
            for (size_t i = 0; i < p->tl_marks.size(); ++i) {
                float ms = 0.f;
                FS_CK(cudaEventElapsedTime(&ms, p->tl_marks[0].second, p->tl_marks[i].second));
                char item[128];
                std::snprintf(item, sizeof item, "%s\"%s\": %.4f", i ? ", " : "",
                              p->tl_marks[i].first.c_str(), ms);
                js += item;
            }
            js += "}";
            if ((int)js.size() + 1 > cap) raise(FS_ERR_CONTRACT, "plan: timeline buffer too small");
            std::memcpy(json, js.c_str(), js.size() + 1);
        } catch (...) {
            cleanup();
            throw;
        }
        cleanup();
    });
}

fs_status fs_plan_timeline_graph(fs_plan p, const uint8_t* const* views_rgba, uint8_t* out_rgba,
                                 void* stream, char* json, int cap) {
    return plan_guard([&] {
        FS_CK(cudaSetDevice(p->device));
        if (!p->dag) raise(FS_ERR_UNSUPPORTED, "plan: timeline needs the DAG schedule");
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        HostIO io{views_rgba, out_rgba};
        if (!p->stamps) FS_CK(cudaMalloc(&p->stamps, sizeof(unsigned long long) * kMaxStamps));
        cudaGraph_t g = nullptr;
        cudaGraphExec_t e = nullptr;
        const int saved = p->launches;
        p->tl_stamp = true;
        p->stamp_labels.clear();
        auto cleanup = [&] {
            p->tl_stamp = false;
            if (e) cudaGraphExecDestroy(e);
            if (g) cudaGraphDestroy(g);
            p->launches = saved;
        };
        try {
            // the production graph with stamp kernels at the schedule points
            capture(p, (views_rgba || out_rgba) ? &io : nullptr, &g, &e);
            for (int rep = 0; rep < 3; ++rep) FS_CK(cudaGraphLaunch(e, s));
            FS_CK(cudaStreamSynchronize(s));
            std::vector<unsigned long long> t(p->stamp_labels.size());
            FS_CK(cudaMemcpy(t.data(), p->stamps, sizeof(unsigned long long) * t.size(),
                             cudaMemcpyDeviceToHost));
            std::string js = "{";
            for (size_t i = 0; i < t.size(); ++i) {
                char item[160];
                std::snprintf(item, sizeof item, "%s\"%s\": %.4f", i ? ", " : "",
                              p->stamp_labels[i].c_str(), (double)(t[i] - t[0]) * 1e-6);
                js += item;
            }
            js += "}";
            if ((int)js.size() + 1 > cap) raise(FS_ERR_CONTRACT, "plan: timeline buffer too small");
            std::memcpy(json, js.c_str(), js.size() + 1);
        } catch (...) {
            cleanup();
            throw;
        }
        cleanup();
    });
}

fs_status fs_plan_profile(fs_plan p, void* stream, fs_kernel_stat* out, int max_out, int* n_out,
                          double* total_ms) {
    return plan_guard([&] {
        FS_CK(cudaSetDevice(p->device));
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        KernelProf prof;
        cudaEvent_t e0, e1;
        FS_CK(cudaEventCreate(&e0));
        FS_CK(cudaEventCreate(&e1));
        kernel_prof() = &prof;
        try {
            FS_CK(cudaEventRecord(e0, s));
            enqueue_all(p, s, false);  // serial, so each kernel is timed alone
            FS_CK(cudaEventRecord(e1, s));
        } catch (...) {
            kernel_prof() = nullptr;
            throw;
        }
        kernel_prof() = nullptr;
        FS_CK(cudaStreamSynchronize(s));
        float tot = 0.f;
        cudaEventElapsedTime(&tot, e0, e1);
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        if (total_ms) *total_ms = tot;
        int n = 0;
        for (auto& r : prof.recs) {
            float ms = 0.f;
            FS_CK(cudaEventElapsedTime(&ms, r.a, r.b));
            int k = 0;
            while (k < n && std::strncmp(out[k].name, r.name, sizeof(out[k].name)) != 0) ++k;
            if (k == n) {
                if (n == max_out) continue;
                std::memset(&out[n], 0, sizeof(out[n]));
                std::strncpy(out[n].name, r.name, sizeof(out[n].name) - 1);
                ++n;
            }
            out[k].launches += 1;
            out[k].ms += ms;
            out[k].bytes += r.bytes;
        }
        *n_out = n;
    });
}

fs_status fs_shard_schedule(int n, const int* boxes, int nranks, int* fold_rank, int* stage,
                            int* n_segments, fs_strip_xfer* xfers, int max_xfers, int* n_xfers) {
    return plan_guard([&] {
        if (n < 2) raise(FS_ERR_CONTRACT, "shard: at least two images required");
        std::vector<Rect> bx(n);
        for (int k = 1; k < n; ++k)
            bx[k] = Rect{boxes[4 * k], boxes[4 * k + 1], boxes[4 * k + 2], boxes[4 * k + 3]};
        std::vector<int> fr(n, -1), stg;
        if (fold_rank)
            for (int k = 1; k < n; ++k) fr[k] = fold_rank[k];
        int nseg = 0;
        std::vector<fs_strip_xfer> xf;
        std::vector<std::vector<char>> needed;
        shard_schedule(n, bx, nranks, fr, stg, nseg, xf, needed);
        if ((int)xf.size() > max_xfers) raise(FS_ERR_CONTRACT, "shard: transfer list too small");
        if (fold_rank)
            for (int k = 0; k < n; ++k) fold_rank[k] = fr[k];
        if (stage)
            for (int k = 0; k < n; ++k) stage[k] = stg[k];
        if (n_segments) *n_segments = nseg;
        for (size_t i = 0; i < xf.size(); ++i) xfers[i] = xf[i];
        if (n_xfers) *n_xfers = (int)xf.size();
    });
}

fs_status fs_plan_shard(fs_plan p, int nranks, int rank, const int* fold_rank) {
    return plan_guard([&] {
        FS_CK(cudaSetDevice(p->device));
        shard_configure(p, nranks, rank, fold_rank);
    });
}

int fs_plan_shard_segments(fs_plan p) { return p ? p->shard.nseg : 0; }

int fs_plan_shard_launch_count(fs_plan p) {
    int n = 0;
    if (p)
        for (int l : p->shard.launches) n += l;
    return n;
}

fs_status fs_plan_shard_xfers(fs_plan p, int segment, fs_strip_xfer* out, int max_out,
                              int* n_out) {
    return plan_guard([&] {
        const auto& S = p->shard;
        int n = 0;
        for (const auto& x : S.xfers)
            if (x.stage == segment && (x.src == S.rank || x.dst == S.rank)) {
                if (n == max_out) raise(FS_ERR_CONTRACT, "shard: transfer list too small");
                out[n++] = x;
            }
        *n_out = n;
    });
}

fs_status fs_plan_strip_buffer(fs_plan p, int fold, void** ptr, size_t* bytes) {
    if (!p || fold < 1 || fold >= p->n) return FS_ERR_CONTRACT;
    const FoldWS<ViewU8>& f = p->folds[fold - 1];
    *ptr = f.blended;
    *bytes = (size_t)f.box.w * f.box.h * sizeof(float4);
    return FS_OK;
}

fs_status fs_plan_shard_execute(fs_plan p, int segment, const uint8_t* const* views_rgba,
                                uint8_t* out_rgba, void* stream) {
    return plan_guard([&] {
        FS_CK(cudaSetDevice(p->device));
        auto& S = p->shard;
        if (segment < 0 || segment >= S.nseg) raise(FS_ERR_CONTRACT, "shard: segment out of range");
        if ((int)S.exec.size() != S.nseg) shard_configure(p, S.nranks, S.rank, S.fold_rank.data());
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        // host buffers the graphs can copy asynchronously are captured into
        // the segments: the views into segment 0 (overlapping the folds), the
        // canvas pieces on rank 0 into the segment after which each is final;
        // pageable buffers are copied around the graphs
        const bool last = segment == S.nseg - 1;
        const uint8_t* const* vin = segment == 0 ? views_rgba : nullptr;
        uint8_t* hout = S.rank == 0 ? out_rgba : nullptr;
        bool async_in = true;
        for (int k = 0; vin && k < p->n; ++k) async_in = async_in && async_copyable(vin[k]);
        const bool async_out = hout && async_copyable(hout);
        if (vin && !async_in) {
            for (int k = 0; k < p->n; ++k) upload_view(p, k, vin[k], s);
            vin = nullptr;
        }
        std::vector<const void*> key;
        for (int k = 0; vin && k < p->n; ++k) key.push_back(vin[k]);
        key.push_back(async_out ? hout : nullptr);
        if (S.hkeys.size() != (size_t)S.nseg) S.hkeys.assign(S.nseg, {});
        if (S.hkeys[segment] != key && S.exec[segment]) {
            cudaGraphExecDestroy(S.exec[segment]);
            cudaGraphDestroy(S.graph[segment]);
            S.exec[segment] = nullptr;
            S.graph[segment] = nullptr;
        }
        if (!S.exec[segment]) {
            HostIO io{vin, async_out ? hout : nullptr};
            capture_shard(p, segment, &io);
            S.hkeys[segment] = key;
        }
        FS_CK(cudaGraphLaunch(S.exec[segment], s));
        if (last && hout && !async_out) download_rect(p, Rect{0, 0, p->cw, p->chh}, hout, s);
    });
}

void fs_plan_destroy(fs_plan p) {
    if (!p) return;
    drop_graph(p);
    free_tiles(p);
    for (auto b : p->branch)
        if (b) cudaStreamDestroy(b);
    for (auto e : p->ev_branch)
        if (e) cudaEventDestroy(e);
    for (auto e : p->ev_compose)
        if (e) cudaEventDestroy(e);
    for (auto e : p->ev_chunk) cudaEventDestroy(e);
    for (auto e : p->ev_copied) cudaEventDestroy(e);
    if (p->xst) cudaStreamDestroy(p->xst);
    for (auto e : p->ev_h2d)
        if (e) cudaEventDestroy(e);
    for (auto e : p->ev_own)
        if (e) cudaEventDestroy(e);
    for (auto e : p->ev_efork)
        if (e) cudaEventDestroy(e);
    for (auto e : p->ev_ejoin)
        if (e) cudaEventDestroy(e);
    for (auto st : p->edt_stream)
        if (st) cudaStreamDestroy(st);
    for (auto st : p->a2_stream)
        if (st) cudaStreamDestroy(st);
    for (auto st : p->tensor_stream)
        if (st) cudaStreamDestroy(st);
    for (auto& f : p->folds) flow_destroy_events(f.flow);
    if (p->own) cudaStreamDestroy(p->own);
    for (auto e : p->ev_a2)
        if (e) cudaEventDestroy(e);
    if (p->d2h_early) cudaStreamDestroy(p->d2h_early);
    if (p->hfill) cudaStreamDestroy(p->hfill);
    if (p->ev_hfill1) cudaEventDestroy(p->ev_hfill1);
    for (cudaEvent_t e : {p->ev_start, p->ev_place, p->ev_out, p->ev_out_early, p->ev_clear})
        if (e) cudaEventDestroy(e);
    if (p->hist) cudaFree(p->hist);
    if (p->h2d) cudaStreamDestroy(p->h2d);
    if (p->d2h) cudaStreamDestroy(p->d2h);
    if (p->arena) cudaFree(p->arena);
    if (p->hstats) cudaFreeHost(p->hstats);
    if (p->stamps) cudaFree(p->stamps);
    if (p->landed) cudaFree(p->landed);
    if (p->stage_in) cudaFree(p->stage_in);
    if (p->stage_out) cudaFree(p->stage_out);
    if (p->shard.ev_seg) cudaEventDestroy(p->shard.ev_seg);
    if (p->shard.ev_hist) cudaEventDestroy(p->shard.ev_hist);
    if (p->shard.ev_segend) cudaEventDestroy(p->shard.ev_segend);
    if (p->shard.ev_place0) cudaEventDestroy(p->shard.ev_place0);
    if (p->shard.ev_d2h) cudaEventDestroy(p->shard.ev_d2h);
    if (p->shard.hist) cudaFree(p->shard.hist);
    if (p->cap) cudaStreamDestroy(p->cap);
    delete p;
}

}  // extern "C"
