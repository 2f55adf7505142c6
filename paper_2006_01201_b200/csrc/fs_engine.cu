// Host orchestration of the B200 flow+blend path (see fs_engine.cuh).
#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdlib>
#include <cstring>

#include "fs_engine.cuh"

namespace fs {

void raise(fs_status code, const std::string& msg) { throw Error{code, msg}; }

std::string& last_error_slot() {
    thread_local std::string msg;
    return msg;
}

KernelProf*& kernel_prof() {
    thread_local KernelProf* p = nullptr;
    return p;
}
KernelProf::~KernelProf() {
    for (auto& r : recs) {
        cudaEventDestroy(r.a);
        cudaEventDestroy(r.b);
    }
}
ProfScope::ProfScope(const char* name, double bytes, cudaStream_t s_) : s(s_) {
    KernelProf* p = kernel_prof();
    on = p != nullptr;
    if (!on) return;
    KernelProf::Rec r{name, bytes, nullptr, nullptr};
    cudaEventCreate(&r.a);
    cudaEventCreate(&r.b);
    cudaEventRecord(r.a, s);
    p->recs.push_back(r);
}
ProfScope::~ProfScope() {
    if (on) cudaEventRecord(kernel_prof()->recs.back().b, s);
}

void cuda_check(cudaError_t e, const char* what) {
    if (e == cudaErrorMemoryAllocation) raise(FS_ERR_OOM, std::string("device allocation failed: ") + what);
    if (e != cudaSuccess) raise(FS_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

// Per device (the current one): is it an sm_100 part?  Checked once per
// device, thread-safe; kernel attributes are applied per device (launch::init).
void ensure_device() {
    static std::atomic<unsigned long long> checked{0}, good{0};
    int n = 0, dev = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n <= 0 || cudaGetDevice(&dev) != cudaSuccess) {
        cudaGetLastError();
        raise(FS_ERR_CUDA, "no sm_100 (B200) CUDA device available; the flow+blend path has no "
                           "CPU fallback");
    }
    once_per_device(checked, [&](int d) {
        int major = 0;
        cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, d);
        cudaGetLastError();
        if (major == 10) good.fetch_or(1ull << (d & 63));
    });
    if (!(good.load() & (1ull << (dev & 63))))
        raise(FS_ERR_CUDA, "CUDA device " + std::to_string(dev) + " is not an sm_100 (B200) "
                           "part; the flow+blend path has no CPU fallback");
    launch::init();
}

void check_edt_extent(long long w, long long h, const char* what) {
    if ((w - 1) * (w - 1) + (h - 1) * (h - 1) >= (long long)kInfSq)
        raise(FS_ERR_UNSUPPORTED, std::string(what) + ": a " + std::to_string(w) + "x" +
                                      std::to_string(h) + " canvas exceeds the distance "
                                      "transform's exact range ((w-1)^2 + (h-1)^2 < 2^30 - 1)");
}

// src/flow.cpp:15-21 (same messages)
void validate_flow_params(const fs_flow_params& p) {
    if (p.levels < 1) raise(FS_ERR_CONTRACT, "FlowParams: levels must be >= 1");
    if (p.window_radius < 1) raise(FS_ERR_CONTRACT, "FlowParams: window_radius must be >= 1");
    if (p.iterations_per_level < 1)
        raise(FS_ERR_CONTRACT, "FlowParams: iterations_per_level must be >= 1");
    if (!(p.min_eigen_eps > 0.0)) raise(FS_ERR_CONTRACT, "FlowParams: min_eigen_eps must be > 0");
    if (p.smoothing_passes < 0) raise(FS_ERR_CONTRACT, "FlowParams: smoothing_passes must be >= 0");
    if (p.window_radius > launch::lk_max_radius())
        raise(FS_ERR_UNSUPPORTED, "FlowParams: window_radius above the kernel's maximum (" +
                                      std::to_string(launch::lk_max_radius()) + ")");
}

// src/blender.cpp:11-16
void validate_blend_params(const fs_blend_params& p) {
    if (!(p.k_softmax_sharpness > 0.0) || !std::isfinite(p.k_softmax_sharpness))
        raise(FS_ERR_CONTRACT, "BlendParams: k_softmax_sharpness must be finite and > 0");
    if (p.k_flow_mag_coef < 0.0 || !std::isfinite(p.k_flow_mag_coef))
        raise(FS_ERR_CONTRACT, "BlendParams: k_flow_mag_coef must be finite and >= 0");
}

int pyramid_depth(int w, int h, int levels) {
    int usable = 1;
    while (usable < levels && w / 2 >= 8 && h / 2 >= 8) {
        w /= 2;
        h /= 2;
        ++usable;
    }
    return usable;
}

// ---------------------------------------------------------------------------
void FlowWS::layout(Arena& a, int w_, int h_, int levels, int ndir_) {
    if ((long long)w_ * h_ >= (1LL << 31))
        raise(FS_ERR_UNSUPPORTED, "flow: overlap crops of 2^31 pixels or more are not supported");
    w = w_;
    h = h_;
    ndir = ndir_;
    depth = pyramid_depth(w, h, levels);
    lv.clear();
    int pw = w, ph = h;
    for (int l = 0; l < depth; ++l) {
        lv.push_back({pw, ph});
        pw = std::max(1, pw / 2);
        ph = std::max(1, ph / 2);
    }
    for (int i = 0; i < 2; ++i) {
        pyr[i].assign(depth, nullptr);
        for (int l = 1; l < depth; ++l) pyr[i][l] = a.take<float>((size_t)lv[l].w * lv[l].h);
    }
    size_t n = (size_t)w * h;
    for (int d = 0; d < ndir; ++d) {
        for (int q = 0; q < 2; ++q) {
            fb[d][q] = a.take<float2>(n);
            ok[d][q] = a.take<uint8_t>(n);
        }
        coef[d].assign(depth, nullptr);
        for (int l = 0; l < depth; ++l) coef[d][l] = a.take<float4>((size_t)lv[l].w * lv[l].h);
    }
}

// ---- row/column tiles ------------------------------------------------------
// The dependency cone, walked back from the interior: at level l the
// smoothing passes (1 px each), then every iteration (its outputs need the
// flow and the gathered taps of the pixels within r), then the 2x upsample
// (align-centres bilinear + nearest ever_ok, src/flow.cpp:138-170) into level
// l + 1.  A cut edge of the region clamps the tile's pyramid: level l + 1's
// 5-tap downsample (src/flow.cpp:29-56) reads level l within 2 px, so the
// clamped border grows to c_{l+1} = ceil((c_l + 2) / 2) px; everything the
// interior depends on must stay `m` px inside it (m: room for the taps,
// certified on the device).
static bool tile_certs(int r0, int r1, int i0, int i1, int len, int depth,
                       const fs_flow_params& p, int margin, std::vector<TileCert>& cert) {
    const int R = r1 - r0, N = p.iterations_per_level, r = p.window_radius;
    const bool cut_lo = r0 > 0, cut_hi = r1 < len;
    cert.assign((size_t)depth * N, TileCert{});
    int lo = i0 - r0, hi = i1 - r0, c = 0;
    for (int l = 0; l < depth; ++l) {
        const int n = R >> l;
        // the exact part; a true crop edge clamps like the untiled crop: no bound
        const int exlo = cut_lo ? c : -(1 << 29), exhi = cut_hi ? n - c : (1 << 29);
        const int m = std::max(1, (margin + (1 << l) - 1) >> l);
        lo -= p.smoothing_passes;
        hi += p.smoothing_passes;
        for (int it = N - 1; it >= 0; --it) {
            int zl = lo - r, zh = hi + r;
            if (cut_lo ? zl < exlo + m : false) return false;
            if (cut_hi ? zh > exhi - m : false) return false;
            zl = std::max(zl, 0);
            zh = std::min(zh, n);
            cert[(size_t)l * N + it] = TileCert{zl, zh, exlo, exhi};
            lo = zl;
            hi = zh;
        }
        if (l + 1 < depth) {  // fine u -> coarse (u + 0.5) * 0.5 - 0.5, bilinear + nearest
            lo = std::max(0, (int)std::floor(lo * 0.5 - 0.25));
            hi = std::min(n >> 1, (int)std::floor((hi - 1) * 0.5 - 0.25) + 2);
            c = (c + 3) / 2;
        }
    }
    return true;
}

bool plan_flow_tiles(int w, int h, int axis, int tile_len, int margin, const fs_flow_params& p,
                     std::vector<FlowTile>& tiles) {
    tiles.clear();
    const int len = axis ? h : w;
    const int depth = pyramid_depth(w, h, p.levels);
    const int align = 1 << (depth - 1);
    if (tile_len <= 0 || len % align || len <= tile_len) return false;
    const int nt = (len + tile_len - 1) / tile_len;
    std::vector<int> cuts{0};
    for (int t = 1; t < nt; ++t) {
        const int c = (int)((long long)len * t / nt) / align * align;
        if (c > cuts.back()) cuts.push_back(c);
    }
    cuts.push_back(len);
    if (cuts.size() < 3) return false;
    for (size_t t = 0; t + 1 < cuts.size(); ++t) {
        FlowTile ft;
        ft.axis = axis;
        const int i0 = cuts[t], i1 = cuts[t + 1];
        std::vector<TileCert> cert;
        bool ok = false;
        int r0 = 0, r1 = len;
        for (int H = align; !ok; H += align) {
            r0 = std::max(0, i0 - H);
            r1 = std::min(len, i1 + H);
            ok = tile_certs(r0, r1, i0, i1, len, depth, p, margin, cert);
            if (!ok && r0 == 0 && r1 == len) break;
        }
        const int rw = axis ? w : r1 - r0, rh = axis ? r1 - r0 : h;
        if (!ok || pyramid_depth(rw, rh, p.levels) != depth) {
            tiles.clear();
            return false;
        }
        // test hook (tests/test_gpu_tiles.py): FS_TILE_CERT_SHRINK=k narrows
        // every certified exact part by k px after planning, so the device
        // certificate must refuse the tiles
        if (const char* sh = getenv("FS_TILE_CERT_SHRINK")) {
            const int k = atoi(sh);
            for (TileCert& c : cert) {
                c.exlo += k;
                c.exhi -= k;
            }
        }
        ft.region = axis ? Rect{0, r0, w, r1 - r0} : Rect{r0, 0, r1 - r0, h};
        ft.interior = axis ? Rect{0, i0, w, i1 - i0} : Rect{i0, 0, i1 - i0, h};
        ft.flow.cert = cert;
        ft.flow.cert_axis = axis;
        tiles.push_back(std::move(ft));
    }
    return true;
}

void layout_flow_tile(FlowTile& t, Arena& a, const fs_flow_params& p, int box_w, int box_h) {
    const size_t n = (size_t)t.region.w * t.region.h;
    t.gray[0] = a.take<float>(n);
    t.gray[1] = a.take<float>(n);
    std::vector<TileCert> cert = t.flow.cert;
    const int axis = t.flow.cert_axis;
    t.flow.layout(a, t.region.w, t.region.h, p.levels, 2);
    t.flow.cert = cert;
    t.flow.cert_axis = axis;
    t.flow.cap_lv.clear();
    int pw = box_w, ph = box_h;
    for (int l = 0; l < t.flow.depth; ++l) {
        t.flow.cap_lv.push_back({pw, ph});
        pw = std::max(1, pw / 2);
        ph = std::max(1, ph / 2);
    }
    for (int d = 0; d < 2; ++d) {
        t.vec[d] = a.take<float2>(n);
        t.valid[d] = a.take<uint8_t>(n);
    }
}

void flow_split_events(FlowWS& ws) {
    if (!ws.ev_fork) FS_CK(cudaEventCreateWithFlags(&ws.ev_fork, cudaEventDisableTiming));
    while ((int)ws.ev_tensor.size() < ws.depth) {
        cudaEvent_t e;
        FS_CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        ws.ev_tensor.push_back(e);
    }
}
void flow_destroy_events(FlowWS& ws) {
    if (ws.ev_fork) cudaEventDestroy(ws.ev_fork);
    for (auto e : ws.ev_tensor) cudaEventDestroy(e);
    ws.ev_fork = nullptr;
    ws.ev_tensor.clear();
}

int flow_enqueue(FlowWS& ws, const float* g0, const float* g1, const fs_flow_params& p,
                 float2* const out_vec[2], uint8_t* const out_valid[2], cudaStream_t s,
                 cudaStream_t ts) {
    int launches = 0;
    ws.pyr[0][0] = const_cast<float*>(g0);
    ws.pyr[1][0] = const_cast<float*>(g1);
    for (int l = 1; l < ws.depth; ++l) {
        // read level l-1 once, write level l: (4 n_{l-1} + 4 n_l) per image
        double bytes = 2.0 * 4.0 * ((double)ws.lv[l - 1].w * ws.lv[l - 1].h +
                                    (double)ws.lv[l].w * ws.lv[l].h);
        ProfScope ps("pyramid", bytes, s);
        launch::downsample(ws.pyr[0][l - 1], ws.pyr[1][l - 1], ws.pyr[0][l], ws.pyr[1][l],
                           ws.lv[l - 1].w, ws.lv[l - 1].h, 2, s);
        ++launches;
    }
    const int r = p.window_radius;
    const double win_area = static_cast<double>(2 * r + 1) * (2 * r + 1);
    const double eig_thresh = p.min_eigen_eps * win_area;  // src/flow.cpp:205-206
    static const char* kSweepNames[3][8] = {
        {"lk_iter", "lk_iter_L1", "lk_iter_L2", "lk_iter_L3", "lk_iter_L4", "lk_iter_L5",
         "lk_iter_L6", "lk_iter_L7"},
        {"lk_first", "lk_first_L1", "lk_first_L2", "lk_first_L3", "lk_first_L4",
         "lk_first_L5", "lk_first_L6", "lk_first_L7"},
        {"lk_tensor", "lk_tensor_L1", "lk_tensor_L2", "lk_tensor_L3", "lk_tensor_L4",
         "lk_tensor_L5", "lk_tensor_L6", "lk_tensor_L7"}};
    auto level_args = [&](int l) {
        const Level L = ws.lv[l];
        LkArgs a{};
        a.ndir = ws.ndir;
        a.w = L.w;
        a.h = L.h;
        a.r = r;
        a.th = 0;  // per-level choice (launch::lk_tile_rows)
// coarse levels run while other folds' kernels hold most of the GPU (the
// folds of a phase start together, and the level tensors run beside the
// chain): their tile height is chosen for a third of the CTA slots, i.e.
// taller tiles, less halo work (C2 3.47 -> 3.42 ms, C4 7.70 -> 7.51 ms);
// level 0 keeps the whole-GPU choice
#ifndef LK_COARSE_SLOT_DIV
#define LK_COARSE_SLOT_DIV 3
#endif
        a.slot_div = l >= 1 ? LK_COARSE_SLOT_DIV : 1;
        a.eig_thresh = eig_thresh;
        // src/flow.cpp:241 (a tile: the whole crop's level)
        const Level C = ws.cap_lv.empty() ? L : ws.cap_lv[l];
        a.flow_cap = static_cast<float>(std::max(C.w, C.h));
        a.cert_fail = nullptr;
        for (int d = 0; d < ws.ndir; ++d) {
            int src = ws.ndir == 1 ? 0 : d;
            a.d[d].F = ws.pyr[src][l];
            a.d[d].T = ws.pyr[1 - src][l];
            a.d[d].coef = ws.coef[d][l];
        }
        return a;
    };
    // split schedule: the structure tensors need only the pyramid (the level's
    // `from` gradients), so they run on ts while the chain works coarse to fine
    const bool split = ts && ws.ev_fork && (int)ws.ev_tensor.size() >= ws.depth;
    const bool certify = ws.cert_fail && !ws.cert.empty();
    if (certify && !split)  // the tap certificate lives in the fp32 FIRST/ITER sweeps
        raise(FS_ERR_UNSUPPORTED, "flow tiles need the split LK schedule");
    if (split) {
        FS_CK(cudaEventRecord(ws.ev_fork, s));
        FS_CK(cudaStreamWaitEvent(ts, ws.ev_fork, 0));
        // the coarsest level's tensor is the chain's first need: on the chain
        // itself when other folds' side work competes for the GPU (see
        // FlowWS::tensor0_on_chain)
        const int l_chain = ws.tensor0_on_chain ? ws.depth - 1 : -1;
        for (int l = ws.depth - 1; l >= 0; --l) {
            LkArgs a = level_args(l);
            cudaStream_t st = l == l_chain ? s : ts;
            {
                // per pixel and direction: F 4 in, coef 16 out
                ProfScope ps(kSweepNames[2][std::min(l, 7)],
                             20.0 * ws.lv[l].w * ws.lv[l].h * ws.ndir, st);
                FS_CK(launch::lk_sweep(a, 2, st));
                if (ws.mark && getenv("FS_TL_FINE")) ws.mark("T" + std::to_string(l), st);
            }
            ++launches;
            FS_CK(cudaEventRecord(ws.ev_tensor[l], st));
        }
    }
    int fcur = 0, okcur = 0;
    for (int l = ws.depth - 1; l >= 0; --l) {
        if (ws.mark) ws.mark("L" + std::to_string(l), s);
        const Level L = ws.lv[l];
        const double npx = (double)L.w * L.h * ws.ndir;
        LkArgs a = level_args(l);
        a.mode = l == ws.depth - 1 ? 0 : 2;
        if (a.mode == 2) {
            a.cw = ws.lv[l + 1].w;
            a.ch = ws.lv[l + 1].h;
            a.sx = static_cast<double>(a.cw) / L.w;  // src/flow.cpp:145-146
            a.sy = static_cast<double>(a.ch) / L.h;
        }
        if (!split && p.iterations_per_level == 1)
            for (int d = 0; d < ws.ndir; ++d) a.d[d].coef = nullptr;  // FULL alone: not stored
        // level start: flow (zero / upsampled), ever_ok, It
        for (int d = 0; d < ws.ndir; ++d) {
            a.d[d].fin = ws.fb[d][fcur];
            a.d[d].okin = ws.ok[d][okcur];
            a.d[d].fout = ws.fb[d][fcur ^ 1];
            a.d[d].okout = ws.ok[d][okcur ^ 1];
        }
        {
            // flow 8 + ok 1 out, + the coarser flow/ok 9/4
            ProfScope ps("lk_prep", (9.0 + (a.mode == 2 ? 2.25 : 0.0)) * npx, s);
            FS_CK(launch::lk_prep(a, s));
            if (ws.mark && getenv("FS_TL_FINE")) ws.mark("L" + std::to_string(l) + "_prep", s);
        }
        ++launches;
        fcur ^= 1;
        okcur ^= 1;
        for (int it = 0; it < p.iterations_per_level; ++it) {
            const bool full = it == 0;
            for (int d = 0; d < ws.ndir; ++d) {
                a.d[d].fin = ws.fb[d][fcur];
                a.d[d].okin = ws.ok[d][okcur];
                a.d[d].fout = ws.fb[d][fcur ^ 1];
                a.d[d].okout = ws.ok[d][okcur ^ 1];
            }
            if (full && split) FS_CK(cudaStreamWaitEvent(s, ws.ev_tensor[l], 0));
            if (certify) {
                const TileCert& c = ws.cert[(size_t)l * p.iterations_per_level + it];
                a.cert_fail = ws.cert_fail;
                a.cert_axis = ws.cert_axis;
                a.zlo = c.zlo;
                a.zhi = c.zhi;
                a.exlo = c.exlo;
                a.exhi = c.exhi;
            }
            {
                // 26 B per px, direction and iteration
                // (F 4 + T 4 + flow r/w 16 + ok r/w 2); the level-constant
                // inverse tensor this design also moves (16 B) is not counted
                ProfScope ps(kSweepNames[full && !split][std::min(l, 7)], 26.0 * npx, s);
                FS_CK(launch::lk_sweep(a, full ? (split ? 3 : 1) : 0, s));
                if (ws.mark && getenv("FS_TL_FINE"))
                    ws.mark("L" + std::to_string(l) + "_it" + std::to_string(it), s);
            }
            ++launches;
            fcur ^= 1;
            if (full) okcur ^= 1;  // ever_ok is final after a level's first iteration
        }
        int P = p.smoothing_passes;
        while (P > 0) {
            int passes = std::min(2, P);
            P -= passes;
            bool fin = (l == 0 && P == 0);
            SmoothArgs a{};
            a.ndir = ws.ndir;
            a.w = L.w;
            a.h = L.h;
            a.passes = passes;
            a.final_cap = fin ? static_cast<float>(ws.cap_lv.empty() ? std::max(ws.w, ws.h)
                                                                     : std::max(ws.cap_lv[0].w,
                                                                                ws.cap_lv[0].h))
                              : 0.f;
            for (int d = 0; d < ws.ndir; ++d) {
                a.fin[d] = ws.fb[d][fcur];
                a.fout[d] = fin ? out_vec[d] : ws.fb[d][fcur ^ 1];
                a.ok[d] = ws.ok[d][okcur];
                a.valid_out[d] = out_valid[d];
            }
            {
                // 16 B per px, direction and pass
                ProfScope ps(l == 0 ? "smooth" : "smooth_coarse",
                             16.0 * passes * L.w * L.h * ws.ndir, s);
                launch::smooth(a, s);
            }
            ++launches;
            if (!fin) fcur ^= 1;
        }
        if (l == 0 && p.smoothing_passes == 0) {
            SmoothArgs a{};
            a.ndir = ws.ndir;
            a.w = L.w;
            a.h = L.h;
            a.final_cap = static_cast<float>(
                ws.cap_lv.empty() ? std::max(ws.w, ws.h)
                                  : std::max(ws.cap_lv[0].w, ws.cap_lv[0].h));
            for (int d = 0; d < ws.ndir; ++d) {
                a.fin[d] = ws.fb[d][fcur];
                a.fout[d] = out_vec[d];
                a.ok[d] = ws.ok[d][okcur];
                a.valid_out[d] = out_valid[d];
            }
            {
                ProfScope ps("smooth", 18.0 * L.w * L.h * ws.ndir, s);
                launch::finalize_flow(a, s);
            }
            ++launches;
        }
    }
    if (ws.mark) ws.mark("flow_end", s);
    FS_CK(cudaGetLastError());
    return launches;
}

// ---------------------------------------------------------------------------
static Rect intersect(const Rect& a, const Rect& b) {
    int x0 = std::max(a.x0, b.x0), y0 = std::max(a.y0, b.y0);
    int x1 = std::min(a.x1(), b.x1()), y1 = std::min(a.y1(), b.y1());
    Rect r;
    r.x0 = x0;
    r.y0 = y0;
    r.w = std::max(0, x1 - x0);
    r.h = std::max(0, y1 - y0);
    return r;
}

EdtPlan edt_plan(const Rect& C, const Rect& E, bool full_domain) {
    EdtPlan p;
    p.C = C;
    p.E = E;
    p.vfirst = C.h >= C.w ? 1 : 0;
    if (full_domain) {
        p.W = E;
        return p;
    }
    int M = std::min(C.w, C.h) + 8;
    Rect grown;
    grown.x0 = C.x0 - M;
    grown.y0 = C.y0 - M;
    grown.w = C.w + 2 * M;
    grown.h = C.h + 2 * M;
    p.W = intersect(grown, E);
    p.e_left = p.W.x0 == E.x0;
    p.e_right = p.W.x1() == E.x1();
    p.e_top = p.W.y0 == E.y0;
    p.e_bottom = p.W.y1() == E.y1();
    p.check = !(p.e_left && p.e_right && p.e_top && p.e_bottom);
    return p;
}

void EdtWS::layout(Arena& a, const Rect& C, const Rect& E) {
    bool vfirst = C.h >= C.w;
    size_t gsz = vfirst ? (size_t)C.h * E.w : (size_t)C.w * E.h;
    size_t nlines = vfirst ? E.w : E.h;
    size_t nseg = ((vfirst ? E.h : E.w) + 63) / 64;
    g = a.take<int>(gsz);
    stack = a.take<int>(gsz);
    bits = a.take<unsigned long long>(nlines * nseg);
    out = a.take<int>((size_t)C.w * C.h);
}

template <class V>
void FoldWS<V>::layout(Arena& a, const Rect& box_, const Rect& pano_bbox, const Rect& view_rect,
                       const fs_flow_params& fp) {
    box = box_;
    E1 = pano_bbox;
    E2 = view_rect;
    size_t n = (size_t)box.w * box.h;
    gray[0] = a.take<float>(n);
    gray[1] = a.take<float>(n);
    flow.layout(a, box.w, box.h, fp.levels, 2);
    depth = flow.depth;
    for (int d = 0; d < 2; ++d) {
        fvec[d] = a.take<float2>(n);
        fvalid[d] = a.take<uint8_t>(n);
    }
    edt[0].layout(a, box, E1);
    edt[1].layout(a, box, E2);
    blended = a.take<float4>(n);
    st = a.take<FoldStats>(1);
    replan_edt();
}

template <class V>
void FoldWS<V>::replan_edt() {
    ep[0] = edt_plan(box, E1, full_domain);
    ep[1] = edt_plan(box, E2, full_domain);
}

__global__ void k_init_stats(FoldStats* st) {
    st->cnt2 = 0;
    st->cnt3 = 0;
    st->bx0 = INT_MAX;
    st->by0 = INT_MAX;
    st->bx1 = -1;
    st->by1 = -1;
    st->edt_fail = 0;
    st->box_mismatch = 0;
    st->reach_fail = 0;
    st->tile_fail = 0;
}
__global__ void k_init_count(CanvasCount* cc) { cc->valid_count = 0; }

void init_stats(FoldStats* st, cudaStream_t s) { k_init_stats<<<1, 1, 0, s>>>(st); }
void init_count(CanvasCount* cc, cudaStream_t s) { k_init_count<<<1, 1, 0, s>>>(cc); }

template <class V, class P>
int fold_enqueue_pre(FoldWS<V>& f, const P& pano, const V& view, cudaStream_t s) {
    init_stats(f.st, s);
    {
        ProfScope ps("partition", 5.0 * view.rect.area(), s);  // view 4 B + pano valid 1 B
        launch::partition(pano, view, f.st, s);
    }
    return 2;
}

template <class V, class P, class PC>
int fold_enqueue_flow_edt(FoldWS<V>& f, const P& pano, const PC& crop_src, const V& view, int ch,
                          const fs_flow_params& fp, cudaStream_t s, cudaEvent_t ev_flow0,
                          cudaEvent_t ev_flow1, cudaStream_t es, cudaEvent_t ev_fork,
                          cudaEvent_t ev_join, bool with_edt, cudaStream_t ts,
                          cudaEvent_t ev_data) {
    int launches = 0;
    // the distance transforms need only the masks and the fold's counts: with
    // a second stream they run concurrently with the flow
    cudaStream_t se = s;
    if (!with_edt) es = nullptr;
    if (es) {
        FS_CK(cudaEventRecord(ev_fork, s));
        FS_CK(cudaStreamWaitEvent(es, ev_fork, 0));
        se = es;
    }
    if (ev_data) FS_CK(cudaStreamWaitEvent(s, ev_data, 0));  // the crop's pixels landed
    launch::check_box(f.st, f.box, s);
    {
        // pano rgb 16 + valid 1 + view 4 in, two gray planes 8 out
        ProfScope ps("crop_gray", 29.0 * f.box.area(), s);
        launch::crop_gray(crop_src, view, f.box, ch, f.gray[0], f.gray[1], s);
    }
    launches += 2;
    if (ev_flow0) FS_CK(cudaEventRecord(ev_flow0, s));
    if (es) launches += fold_enqueue_edt(f, pano, view, se);
    launches += flow_enqueue(f.flow, f.gray[0], f.gray[1], fp, f.fvec, f.fvalid, s, ts);
    if (ev_flow1) FS_CK(cudaEventRecord(ev_flow1, s));
    if (es) {
        FS_CK(cudaEventRecord(ev_join, es));
        FS_CK(cudaStreamWaitEvent(s, ev_join, 0));
    } else if (with_edt) {
        launches += fold_enqueue_edt(f, pano, view, s);
    }
    FS_CK(cudaGetLastError());
    return launches;
}

template <class V, class P>
int fold_enqueue_edt(FoldWS<V>& f, const P& pano, const V& view, cudaStream_t s) {
    EdtJob<FoldMask<V, P>> j[2];
    for (int m = 0; m < 2; ++m) {
        const EdtPlan& E = f.ep[m];
        j[m].mask = FoldMask<V, P>{pano, view, m + 1};
        j[m].which = m + 1;
        j[m].active = 1;
        j[m].W = E.W;
        j[m].C = E.C;
        j[m].vfirst = E.vfirst;
        j[m].g = f.edt[m].g;
        j[m].bits = f.edt[m].bits;
        j[m].stack = f.edt[m].stack;
        j[m].out = f.edt[m].out;
        j[m].e_left = E.e_left;
        j[m].e_right = E.e_right;
        j[m].e_top = E.e_top;
        j[m].e_bottom = E.e_bottom;
        j[m].check = E.check;
    }
    {
        // per mask: the seed mask over the domain (pano valid 1 + view 4) + d^2 out on C
        double bytes = 0;
        for (int m = 0; m < 2; ++m) bytes += 5.0 * f.ep[m].W.area() + 4.0 * f.box.area();
        ProfScope ps("edt", bytes, s);
        launch::edt(j[0], j[1], f.st, s);
    }
    return 3;
}

template <class V>
int fold_enqueue_blend(FoldWS<V>& f, const Canvas& cv, const V& view, CanvasCount* cc,
                       const fs_blend_params& bp, cudaStream_t s, const uint8_t* owner, int fold,
                       uchar4* out, const ReachCheck* rc, const PanoViews* first_cover,
                       bool write_cv) {
    int launches = 0;
    // no later fold reads this fold's blended pixels (write_cv false): the
    // blend writes the RGBA8 canvas itself and there is no compose
    const bool direct = owner && out && !write_cv;
    {
        // pano rgb 16 + valid 1, view 4, two flows 16, two d^2 8 in; 16 out
        ProfScope ps("blend", 61.0 * f.box.area(), s);
        launch::blend_area3(cv, view, f.box, f.fvec[0], f.fvec[1], f.edt[0].out, f.edt[1].out,
                            f.st, bp.k_softmax_sharpness, bp.k_flow_mag_coef, f.blended, f.wgray,
                            owner, fold, s, rc, first_cover, direct ? out : nullptr);
    }
    if (direct) {
        FS_CK(cudaGetLastError());
        return launches + 1;
    }
    if (owner) {  // Area3 only: the fold's Area2 was copied on its branch
        ProfScope ps("compose", 21.0 * f.box.area(), s);  // owner 1 + view 4 + blended 16
        launch::compose_area3(cv, view, f.box, f.blended, owner, fold, s, out, write_cv);
        FS_CK(cudaGetLastError());
        return launches + 2;
    }
    {
        // view 4 + pano valid 1 in, rgb 16 + valid 1 out on the view; blended 16 in on Area3
        ProfScope ps("compose", 22.0 * view.rect.area() + 16.0 * f.box.area(), s);
        launch::compose(cv, view, f.box, f.blended, cc, f.st, s);
    }
    launches += 3;
    FS_CK(cudaGetLastError());
    return launches;
}

template struct FoldWS<ViewU8>;
template struct FoldWS<ViewF4>;
template int fold_enqueue_pre<ViewU8, PanoViews>(FoldWS<ViewU8>&, const PanoViews&, const ViewU8&,
                                                 cudaStream_t);
template int fold_enqueue_pre<ViewU8, PanoPlane>(FoldWS<ViewU8>&, const PanoPlane&, const ViewU8&,
                                                 cudaStream_t);
template int fold_enqueue_pre<ViewF4, PanoPlane>(FoldWS<ViewF4>&, const PanoPlane&, const ViewF4&,
                                                 cudaStream_t);
template int fold_enqueue_flow_edt<ViewU8, PanoViews, PanoViews>(
    FoldWS<ViewU8>&, const PanoViews&, const PanoViews&, const ViewU8&, int,
    const fs_flow_params&, cudaStream_t, cudaEvent_t, cudaEvent_t, cudaStream_t,
    cudaEvent_t, cudaEvent_t, bool, cudaStream_t, cudaEvent_t);
template int fold_enqueue_flow_edt<ViewU8, PanoViews, PanoHybrid>(
    FoldWS<ViewU8>&, const PanoViews&, const PanoHybrid&, const ViewU8&, int,
    const fs_flow_params&, cudaStream_t, cudaEvent_t, cudaEvent_t, cudaStream_t,
    cudaEvent_t, cudaEvent_t, bool, cudaStream_t, cudaEvent_t);
template int fold_enqueue_flow_edt<ViewU8, PanoPlane, PanoPlane>(
    FoldWS<ViewU8>&, const PanoPlane&, const PanoPlane&, const ViewU8&, int,
    const fs_flow_params&, cudaStream_t, cudaEvent_t, cudaEvent_t, cudaStream_t,
    cudaEvent_t, cudaEvent_t, bool, cudaStream_t, cudaEvent_t);
template int fold_enqueue_flow_edt<ViewF4, PanoPlane, PanoPlane>(
    FoldWS<ViewF4>&, const PanoPlane&, const PanoPlane&, const ViewF4&, int,
    const fs_flow_params&, cudaStream_t, cudaEvent_t, cudaEvent_t, cudaStream_t,
    cudaEvent_t, cudaEvent_t, bool, cudaStream_t, cudaEvent_t);
template int fold_enqueue_edt<ViewU8, PanoViews>(FoldWS<ViewU8>&, const PanoViews&, const ViewU8&,
                                                 cudaStream_t);
template int fold_enqueue_blend<ViewU8>(FoldWS<ViewU8>&, const Canvas&, const ViewU8&,
                                        CanvasCount*, const fs_blend_params&, cudaStream_t,
                                        const uint8_t*, int, uchar4*, const ReachCheck*,
                                        const PanoViews*, bool);
template int fold_enqueue_blend<ViewF4>(FoldWS<ViewF4>&, const Canvas&, const ViewF4&,
                                        CanvasCount*, const fs_blend_params&, cudaStream_t,
                                        const uint8_t*, int, uchar4*, const ReachCheck*,
                                        const PanoViews*, bool);

}  // namespace fs
