// Planned, graph-captured fold over 8-bit views (the production path of
// include/fs_b200.h).  A plan fixes the layout and owns every device buffer;
// one execution is a single CUDA-graph launch that recomputes the whole fold
// (partition, crop+gray, pyramid, bidirectional LK, distance transforms,
// Code 1 blend, composition, 8-bit quantisation) from the views in HBM.
#include <algorithm>
#include <climits>
#include <cstring>
#include <string>
#include <vector>

#include "fs_engine.cuh"

using namespace fs;

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
    // stream; crop_from_views[k]: fold k's L crop can be read from the views.
    bool dag = false;
    std::vector<cudaStream_t> branch;
    std::vector<cudaEvent_t> ev_branch, ev_compose;
    cudaEvent_t ev_pro = nullptr;
    std::vector<char> crop_from_views;
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
Rect rect_inter(const Rect& a, const Rect& b) {
    int x0 = std::max(a.x0, b.x0), y0 = std::max(a.y0, b.y0);
    int x1 = std::min(a.x1(), b.x1()), y1 = std::min(a.y1(), b.y1());
    return Rect{x0, y0, std::max(0, x1 - x0), std::max(0, y1 - y0)};
}

ViewU8 view_of(const fs_plan_s* p, int k) { return ViewU8{p->views[k], p->rects[k]}; }

PanoViews views_before(const fs_plan_s* p, int k) {
    PanoViews pv{};
    pv.n = k;
    for (int m = 0; m < k; ++m) pv.v[m] = view_of(p, m);
    return pv;
}

// Enqueue one full execution on stream s (captured into the graph).  With
// dag, each fold's partition / crop / pyramid / flow / distance transforms
// run on its own branch stream as soon as their inputs exist, and only the
// blend + compose of the folds form an ordered chain on s.
int enqueue_all(fs_plan_s* p, cudaStream_t s, bool dag) {
    int launches = 0;
    const PanoPlane plane{p->cv.valid, p->cv.rgb, p->cv.w};
    {
        ProfScope ps("clear", (double)p->cw * p->chh, s);
        FS_CK(cudaMemsetAsync(p->cv.valid, 0, (size_t)p->cw * p->chh, s));
    }
    init_count(p->cc, s);
    {
        ProfScope ps("place", 21.0 * p->rects[0].area(), s);  // view 4 in, rgb 16 + valid 1 out
        launch::place_view(p->cv, view_of(p, 0), p->cc, s);
    }
    launches += 2;
    if (!dag) {
        for (int k = 1; k < p->n; ++k) {
            FoldWS<ViewU8>& f = p->folds[k - 1];
            ViewU8 v = view_of(p, k);
            launches += fold_enqueue_pre(f, plane, v, s);
            launch::snapshot_count(f.st, p->cc, s);
            launches += 1 + fold_enqueue_flow_edt(f, plane, plane, v, 3, p->fp, s, nullptr, nullptr);
            launches += fold_enqueue_blend(f, p->cv, v, p->cc, p->bp, s);
        }
    } else {
        // prologue: every fold's partition from the union of the earlier views
        std::vector<FoldStats*> sts;
        for (int k = 1; k < p->n; ++k) {
            launches += fold_enqueue_pre(p->folds[k - 1], views_before(p, k), view_of(p, k), s);
            sts.push_back(p->folds[k - 1].st);
        }
        launch::prefix_counts(sts.data(), (int)sts.size(), p->cc, s);
        ++launches;
        FS_CK(cudaEventRecord(p->ev_pro, s));
        for (int k = 1; k < p->n; ++k) {
            FoldWS<ViewU8>& f = p->folds[k - 1];
            ViewU8 v = view_of(p, k);
            cudaStream_t b = p->branch[k - 1];
            FS_CK(cudaStreamWaitEvent(b, p->ev_pro, 0));
            const PanoViews pv = views_before(p, k);
            if (p->crop_from_views[k]) {
                launches += fold_enqueue_flow_edt(f, pv, pv, v, 3, p->fp, b, nullptr, nullptr);
            } else {  // an earlier Area3 box overlaps: L is the composed panorama
                FS_CK(cudaStreamWaitEvent(b, p->ev_compose[k - 1], 0));
                launches += fold_enqueue_flow_edt(f, pv, plane, v, 3, p->fp, b, nullptr, nullptr);
            }
            FS_CK(cudaEventRecord(p->ev_branch[k], b));
            FS_CK(cudaStreamWaitEvent(s, p->ev_branch[k], 0));
            launches += fold_enqueue_blend(f, p->cv, v, p->cc, p->bp, s);
            FS_CK(cudaEventRecord(p->ev_compose[k], s));
        }
    }
    {
        ProfScope ps("quantize", 21.0 * p->cw * p->chh, s);  // rgb 16 + valid 1 in, rgba8 out
        launch::quantize(p->cv, p->out, s);
    }
    launches += 1;
    FS_CK(cudaGetLastError());
    return launches;
}

void build_graph(fs_plan_s* p) {
    if (p->exec) return;
    FS_CK(cudaStreamBeginCapture(p->cap, cudaStreamCaptureModeThreadLocal));
    int launches = 0;
    try {
        launches = enqueue_all(p, p->cap, p->dag);
    } catch (...) {
        cudaGraph_t g;
        cudaStreamEndCapture(p->cap, &g);
        if (g) cudaGraphDestroy(g);
        throw;
    }
    FS_CK(cudaStreamEndCapture(p->cap, &p->graph));
    FS_CK(cudaGraphInstantiate(&p->exec, p->graph, 0));
    p->launches = launches;
}

void drop_graph(fs_plan_s* p) {
    if (p->exec) cudaGraphExecDestroy(p->exec);
    if (p->graph) cudaGraphDestroy(p->graph);
    p->exec = nullptr;
    p->graph = nullptr;
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
        FS_CK(cudaStreamCreateWithFlags(&p->cap, cudaStreamNonBlocking));
        std::vector<Rect> boxes = views_rgba ? boxes_from_masks(p, views_rgba) : boxes_from_rects(p);
        // DAG: fold k's L crop may come straight from the views when no earlier
        // fold's Area3 box overlaps its own (those pixels hold the first
        // covering view's value); partitions and distance transforms always can.
        p->dag = n <= kMaxDagViews;
        p->crop_from_views.assign(n, 0);
        for (int k = 1; k < n; ++k) {
            bool disjoint = true;
            for (int m = 1; m < k; ++m) {
                Rect i = rect_inter(boxes[m], boxes[k]);
                if (i.w > 0 && i.h > 0) disjoint = false;
            }
            p->crop_from_views[k] = disjoint;
        }
        if (p->dag) {
            p->branch.assign(n - 1, nullptr);
            p->ev_branch.assign(n, nullptr);
            p->ev_compose.assign(n, nullptr);
            for (auto& b : p->branch) FS_CK(cudaStreamCreateWithFlags(&b, cudaStreamNonBlocking));
            for (int k = 0; k < n; ++k) {
                FS_CK(cudaEventCreateWithFlags(&p->ev_branch[k], cudaEventDisableTiming));
                FS_CK(cudaEventCreateWithFlags(&p->ev_compose[k], cudaEventDisableTiming));
            }
            FS_CK(cudaEventCreateWithFlags(&p->ev_pro, cudaEventDisableTiming));
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
        Arena a1;
        a1.base = p->arena;
        layout_plan(p, a1, boxes);
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
        std::vector<FoldStats> hs(p->folds.size());
        for (size_t k = 0; k < p->folds.size(); ++k)
            FS_CK(cudaMemcpy(&hs[k], p->folds[k].st, sizeof(FoldStats), cudaMemcpyDeviceToHost));
        for (size_t k = 0; k < hs.size(); ++k)
            if (hs[k].box_mismatch)
                raise(FS_ERR_CONTRACT, "plan: the views' masks no longer produce the planned "
                                       "overlap of fold #" + std::to_string(k + 1));
        bool widened = false;
        for (size_t k = 0; k < hs.size(); ++k)
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
        if (views_rgba)
            for (int k = 0; k < p->n; ++k)
                FS_CK(cudaMemcpyAsync(p->views[k], views_rgba[k],
                                      (size_t)p->rects[k].w * p->rects[k].h * 4, cudaMemcpyDefault,
                                      s));
        for (int attempt = 0; attempt < 2; ++attempt) {
            build_graph(p);
            FS_CK(cudaGraphLaunch(p->exec, s));
            if (out_rgba)
                FS_CK(cudaMemcpyAsync(out_rgba, p->out, (size_t)p->cw * p->chh * 4,
                                      cudaMemcpyDefault, s));
            FS_CK(cudaStreamSynchronize(s));
            fs_status c = fs_plan_check(p);
            if (c == FS_OK) return;
            if (attempt == 1 || p->exec) raise(c, last_error_slot());
        }
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

void fs_plan_destroy(fs_plan p) {
    if (!p) return;
    drop_graph(p);
    for (auto b : p->branch)
        if (b) cudaStreamDestroy(b);
    for (auto e : p->ev_branch)
        if (e) cudaEventDestroy(e);
    for (auto e : p->ev_compose)
        if (e) cudaEventDestroy(e);
    if (p->ev_pro) cudaEventDestroy(p->ev_pro);
    if (p->arena) cudaFree(p->arena);
    if (p->cap) cudaStreamDestroy(p->cap);
    delete p;
}

}  // extern "C"
