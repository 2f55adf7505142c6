// extern "C" boundary of the B200 flow+blend path (include/fs_b200.h).
// Each entry point validates like the reference function it replaces, stages
// host buffers through the device, runs the sm_100a kernels and maps failures
// to a status code + thread-local message.
#include <algorithm>
#include <climits>
#include <cstring>
#include <memory>
#include <new>
#include <string>
#include <vector>

#include "fs_api_kernels.cuh"
#include "fs_metrics.cuh"
#include "fs_engine.cuh"

using namespace fs;

namespace {

int g_threads = 0;

template <class F>
fs_status guarded(F&& fn) {
    try {
        fn();
        return FS_OK;
    } catch (const Error& e) {
        last_error_slot() = e.msg;
        return e.code;
    } catch (const std::bad_alloc&) {
        last_error_slot() = "host allocation failed";
        return FS_ERR_OOM;
    }
}

bool is_device_ptr(const void* p) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

// Per-call staging of caller buffers (host or device) on one stream.
struct Stage {
    cudaStream_t s;
    std::vector<void*> allocs;
    struct Back {
        void* host;
        const void* dev;
        size_t n;
    };
    std::vector<Back> backs;
    explicit Stage(void* stream) : s(static_cast<cudaStream_t>(stream)) { ensure_device(); }
    ~Stage() {
        for (void* p : allocs) cudaFreeAsync(p, s);
    }
    void* alloc(size_t n) {
        void* p = nullptr;
        FS_CK(cudaMallocAsync(&p, n ? n : 1, s));
        allocs.push_back(p);
        return p;
    }
    template <class T>
    T* tmp(size_t count) {
        return static_cast<T*>(alloc(count * sizeof(T)));
    }
    template <class T>
    const T* in(const T* p, size_t count) {
        if (!p) return nullptr;
        if (is_device_ptr(p)) return p;
        T* d = tmp<T>(count);
        FS_CK(cudaMemcpyAsync(d, p, count * sizeof(T), cudaMemcpyHostToDevice, s));
        return d;
    }
    template <class T>
    T* out(T* p, size_t count) {
        if (!p) return nullptr;
        if (is_device_ptr(p)) return p;
        T* d = tmp<T>(count);
        backs.push_back({p, d, count * sizeof(T)});
        return d;
    }
    template <class T>
    void read(T* host, const T* dev, size_t count) {
        FS_CK(cudaMemcpyAsync(host, dev, count * sizeof(T), cudaMemcpyDeviceToHost, s));
        FS_CK(cudaStreamSynchronize(s));
    }
    void finish() {
        for (auto& b : backs)
            FS_CK(cudaMemcpyAsync(b.host, b.dev, b.n, cudaMemcpyDeviceToHost, s));
        if (!backs.empty()) FS_CK(cudaStreamSynchronize(s));
        FS_CK(cudaGetLastError());
    }
};

void read_counts(const int64_t* counts, int64_t out[4]) {
    if (is_device_ptr(counts))
        FS_CK(cudaMemcpy(out, counts, 4 * sizeof(int64_t), cudaMemcpyDeviceToHost));
    else
        std::memcpy(out, counts, 4 * sizeof(int64_t));
}

void check_dims(int w, int h) {
    if (w < 0 || h < 0) raise(FS_ERR_CONTRACT, "negative image dimensions");
}
void check_ch(int ch) {
    if (ch != 1 && ch != 3) raise(FS_ERR_CONTRACT, "ImageBuf: channels must be 1 or 3");
}

// squared-distance field of a label/plane mask over a whole w x h raster
template <class M>
void full_edt(Stage& st, const M& m0, const M* m1, int w, int h, int* out0, int* out1) {
    Rect R{0, 0, w, h};
    EdtJob<M> j[2];
    const M* ms[2] = {&m0, m1};
    int* outs[2] = {out0, out1};
    for (int q = 0; q < 2; ++q) {
        if (!ms[q]) continue;
        EdtWS ws;
        Arena a0;
        ws.layout(a0, R, R);
        Arena a1;
        a1.base = static_cast<char*>(st.alloc(a0.off));
        ws.layout(a1, R, R);
        j[q].mask = *ms[q];
        j[q].which = 0;
        j[q].active = 1;
        j[q].W = R;
        j[q].C = R;
        j[q].vfirst = h >= w;
        j[q].g = ws.g;
        j[q].bits = ws.bits;
        j[q].stack = ws.stack;
        j[q].out = outs[q];
    }
    if (!m1) j[1].active = 0;
    launch::edt(j[0], j[1], nullptr, st.s);
    FS_CK(cudaGetLastError());
}

}  // namespace

// ============================================================================
extern "C" {

const char* fs_last_error(void) { return last_error_slot().c_str(); }
int fs_abi_version(void) { return 2; }

unsigned int fs_debug_check_failures(int reset) {
    try {
        ensure_device();
    } catch (const Error&) {
        return 0;
    }
    return check_failures_lk(reset != 0) + check_failures_kernels(reset != 0) +
           check_failures_plan(reset != 0);
}
void fs_debug_inject(int mode) {
    try {
        ensure_device();
        check_inject_lk(mode);
    } catch (const Error&) {
    }
}
int fs_debug_checks_built(void) {
#ifdef FS_CHECKS
    return 1;
#else
    return 0;
#endif
}

int fs_device_available(void) {
    try {
        ensure_device();
        return 1;
    } catch (const Error&) {
        return 0;
    }
}

void fs_default_flow_params(fs_flow_params* p) {
    p->levels = 4;
    p->window_radius = 8;
    p->iterations_per_level = 3;
    p->min_eigen_eps = 1e-4;
    p->smoothing_passes = 2;
}
void fs_default_blend_params(fs_blend_params* p) {
    p->k_softmax_sharpness = 10.0;
    p->k_flow_mag_coef = 0.05;
}

void fs_set_thread_count(int n) { g_threads = n < 0 ? 0 : n; }
int fs_thread_count(void) { return g_threads; }

// image.hpp:94 / src/image.cpp:70-83
fs_status fs_to_gray(const float* img, int w, int h, int ch, float* out, void* stream) {
    return guarded([&] {
        check_dims(w, h);
        check_ch(ch);
        size_t n = (size_t)w * h;
        Stage st(stream);
        const float* di = st.in(img, n * ch);
        float* dout = st.out(out, n);
        if (n) api::to_gray(di, (int)n, ch, dout, st.s);
        st.finish();
    });
}

// north_star stage 1 (parity unpinned: no reference counterpart)
fs_status fs_remap_rgba8(const uint8_t* src, int sw, int sh, int channels, const float* map_xy,
                         int w, int h, const float* gains3, uint8_t* out_rgba, void* stream) {
    return guarded([&] {
        if (sw <= 0 || sh <= 0 || w < 0 || h < 0 || (channels != 3 && channels != 4))
            raise(FS_ERR_CONTRACT, "remap_rgba8: invalid image or table size");
        float g[3] = {1.f, 1.f, 1.f};
        if (gains3) {  // three floats, host or device
            if (is_device_ptr(gains3))
                FS_CK(cudaMemcpy(g, gains3, sizeof g, cudaMemcpyDeviceToHost));
            else
                std::memcpy(g, gains3, sizeof g);
        }
        if (!(g[0] >= 0.f && g[1] >= 0.f && g[2] >= 0.f))
            raise(FS_ERR_CONTRACT, "remap_rgba8: chromaticity gains must be >= 0");
        const size_t n = (size_t)w * h;
        if (!n) return;
        Stage st(stream);
        launch::remap_rgba8(st.in(src, (size_t)sw * sh * channels), sw, sh, channels,
                            reinterpret_cast<const float2*>(st.in(map_xy, 2 * n)), w, h, g,
                            reinterpret_cast<uchar4*>(st.out(out_rgba, 4 * n)), st.s);
        FS_CK(cudaGetLastError());
        st.finish();
    });
}

fs_status fs_chroma_gains(int n, const uint8_t* const* views_rgba, const int* dims,
                          const int* offsets, int canvas_w, int canvas_h, float* gains,
                          void* stream) {
    return guarded([&] {
        if (n < 1 || n > kMaxDagViews) raise(FS_ERR_UNSUPPORTED, "chroma_gains: 1..16 views");
        if (!views_rgba || !dims || !offsets || !gains || canvas_w <= 0 || canvas_h <= 0)
            raise(FS_ERR_CONTRACT, "chroma_gains: invalid arguments");
        Stage st(stream);
        PanoViews pv{};
        pv.n = n;
        for (int k = 0; k < n; ++k) {
            Rect r{offsets[2 * k], offsets[2 * k + 1], dims[2 * k], dims[2 * k + 1]};
            if (r.w <= 0 || r.h <= 0 || r.x0 < 0 || r.y0 < 0 || r.x1() > canvas_w ||
                r.y1() > canvas_h)
                raise(FS_ERR_LAYOUT, "chroma_gains: view does not fit inside the canvas");
            pv.v[k] = ViewU8{reinterpret_cast<const uchar4*>(st.in(views_rgba[k], r.area() * 4)), r};
        }
        const size_t nc = (size_t)canvas_w * canvas_h;
        uint8_t* owner = st.tmp<uint8_t>(nc + 4);
        unsigned long long* sums = st.tmp<unsigned long long>((size_t)n * kMaxDagViews * 6);
        FS_CK(cudaMemsetAsync(owner, 0xFF, nc + 4, st.s));
        FS_CK(cudaMemsetAsync(sums, 0, sizeof(unsigned long long) * n * kMaxDagViews * 6, st.s));
        for (int k = 0; k < n; ++k) launch::claim_owner(owner, canvas_w, pv.v[k], k, st.s);
        pv.owner = owner;
        pv.w = canvas_w;
        for (int k = 1; k < n; ++k)
            launch::chroma_sums(owner, canvas_w, pv.v[k], pv, k, sums + (size_t)k * kMaxDagViews * 6,
                                st.s);
        FS_CK(cudaGetLastError());
        std::vector<unsigned long long> hs((size_t)n * kMaxDagViews * 6);
        st.read(hs.data(), sums, hs.size());
        std::vector<double> g((size_t)n * 3, 1.0);
        for (int k = 1; k < n; ++k)
            for (int c = 0; c < 3; ++c) {
                double num = 0.0, den = 0.0;
                for (int m = 0; m < k; ++m) {
                    const unsigned long long* b = &hs[((size_t)k * kMaxDagViews + m) * 6];
                    num += g[(size_t)m * 3 + c] * (double)b[c];
                    den += (double)b[3 + c];
                }
                g[(size_t)k * 3 + c] = den > 0.0 ? num / den : 1.0;
            }
        for (size_t i = 0; i < g.size(); ++i) gains[i] = (float)g[i];
        st.finish();
    });
}

// image.hpp:98 / src/image.cpp:85-113
fs_status fs_bilinear_sample(const float* img, const uint8_t* valid, int w, int h, int ch,
                             const double* xy, int n, float* out, void* stream) {
    return guarded([&] {
        check_ch(ch);
        if (w <= 0 || h <= 0) raise(FS_ERR_CONTRACT, "bilinear_sample: empty image");
        if (n <= 0) return;
        Stage st(stream);
        size_t np = (size_t)w * h;
        api::bilinear_batch(st.in(img, np * ch), st.in(valid, np), w, h, ch, st.in(xy, 2 * (size_t)n),
                            n, st.out(out, (size_t)n * ch), st.s);
        st.finish();
    });
}

// image.hpp:100 / src/image.cpp:115-132
fs_status fs_compute_partition(const uint8_t* mask_l, const uint8_t* mask_r, int w, int h,
                               uint8_t* label, int64_t* counts, void* stream) {
    return guarded([&] {
        check_dims(w, h);
        Stage st(stream);
        size_t n = (size_t)w * h;
        auto* dc = st.tmp<unsigned long long>(4);
        auto* box = st.tmp<int>(4);
        FS_CK(cudaMemsetAsync(dc, 0, 4 * sizeof(unsigned long long), st.s));
        FS_CK(cudaMemsetAsync(box, 0, 4 * sizeof(int), st.s));
        if (n)
            api::partition_planes(st.in(mask_l, n), st.in(mask_r, n), w, h, st.out(label, n), dc,
                                  box, st.s);
        unsigned long long hc[4];
        st.read(hc, dc, 4);
        for (int q = 0; q < 4; ++q) counts[q] = (int64_t)hc[q];
        st.finish();
    });
}

// image.hpp:103 / src/image.cpp:134-162
fs_status fs_crop_overlap(const float* img, const uint8_t* valid, int w, int h, int ch,
                          const uint8_t* label, const int64_t* counts, float* out,
                          uint8_t* out_valid, int* box, void* stream) {
    return guarded([&] {
        check_ch(ch);
        int64_t c[4];
        read_counts(counts, c);
        if (c[3] == 0) raise(FS_ERR_EMPTY_REGION, "crop_overlap: no overlap (Area3 is empty)");
        Stage st(stream);
        size_t n = (size_t)w * h;
        const uint8_t* dl = st.in(label, n);
        int* db = st.tmp<int>(4);
        int init[4] = {INT_MAX, INT_MAX, -1, -1};
        FS_CK(cudaMemcpyAsync(db, init, sizeof(init), cudaMemcpyHostToDevice, st.s));
        api::label_box(dl, w, h, db, st.s);
        int hb[4];
        st.read(hb, db, 4);
        if (hb[2] < 0) raise(FS_ERR_EMPTY_REGION, "crop_overlap: no overlap (Area3 is empty)");
        box[0] = hb[0];
        box[1] = hb[1];
        box[2] = hb[2] - hb[0] + 1;
        box[3] = hb[3] - hb[1] + 1;
        if (!out) return;
        size_t nc = (size_t)box[2] * box[3];
        api::crop(st.in(img, n * ch), st.in(valid, n), w, ch, dl, box[0], box[1], box[2], box[3],
                  st.out(out, nc * ch), st.out(out_valid, nc), st.s);
        st.finish();
    });
}

// image.hpp:107-108 / src/image.cpp:164-177
fs_status fs_place_on_canvas(const float* img, const uint8_t* valid, int w, int h, int ch,
                             int offset_x, int offset_y, int canvas_w, int canvas_h, float* out,
                             uint8_t* out_valid, void* stream) {
    return guarded([&] {
        check_ch(ch);
        if (offset_x < 0 || offset_y < 0 || offset_x + w > canvas_w || offset_y + h > canvas_h)
            raise(FS_ERR_LAYOUT, "place_on_canvas: image does not fit inside the canvas");
        Stage st(stream);
        size_t nc = (size_t)canvas_w * canvas_h, n = (size_t)w * h;
        float* dout = st.out(out, nc * ch);
        uint8_t* dv = st.out(out_valid, nc);
        FS_CK(cudaMemsetAsync(dout, 0, nc * ch * sizeof(float), st.s));
        FS_CK(cudaMemsetAsync(dv, 0, nc, st.s));
        if (n)
            api::place(st.in(img, n * ch), st.in(valid, n), w, h, ch, offset_x, offset_y,
                       canvas_w, dout, dv, st.s);
        st.finish();
    });
}

int fs_pyramid_depth(int w, int h, int levels) { return pyramid_depth(w, h, levels); }

// flow.hpp:48 / src/flow.cpp:174-192
fs_status fs_build_pyramid(const float* gray, int w, int h, int levels, float* out, int* depth,
                           void* stream) {
    return guarded([&] {
        if (levels < 1) raise(FS_ERR_CONTRACT, "build_pyramid: levels must be >= 1");
        int d = pyramid_depth(w, h, levels);
        size_t total = 0;
        std::vector<size_t> off;
        int pw = w, ph = h;
        for (int l = 0; l < d; ++l) {
            off.push_back(total);
            total += (size_t)pw * ph;
            pw = std::max(1, pw / 2);
            ph = std::max(1, ph / 2);
        }
        Stage st(stream);
        float* dout = st.out(out, total);
        FS_CK(cudaMemcpyAsync(dout, st.in(gray, (size_t)w * h), (size_t)w * h * sizeof(float),
                              cudaMemcpyDeviceToDevice, st.s));
        pw = w;
        ph = h;
        for (int l = 1; l < d; ++l) {
            launch::downsample(dout + off[l - 1], dout + off[l - 1], dout + off[l], dout + off[l],
                               pw, ph, 1, st.s);
            pw = std::max(1, pw / 2);
            ph = std::max(1, ph / 2);
        }
        if (depth) *depth = d;
        st.finish();
    });
}

namespace {
void run_flow(Stage& st, const float* g0, const float* g1, int w, int h, const fs_flow_params& p,
              int ndir, float* vec0, uint8_t* val0, float* vec1, uint8_t* val1) {
    FlowWS ws;
    Arena a0;
    ws.layout(a0, w, h, p.levels, ndir);
    Arena a1;
    a1.base = static_cast<char*>(st.alloc(a0.off));
    ws.layout(a1, w, h, p.levels, ndir);
    size_t n = (size_t)w * h;
    float2* ov[2] = {reinterpret_cast<float2*>(st.out(vec0, 2 * n)),
                     ndir > 1 ? reinterpret_cast<float2*>(st.out(vec1, 2 * n)) : nullptr};
    uint8_t* oval[2] = {st.out(val0, n), ndir > 1 ? st.out(val1, n) : nullptr};
    flow_enqueue(ws, g0, g1, p, ov, oval, st.s);
}
}  // namespace

// flow.hpp:52 / src/flow.cpp:194-314
fs_status fs_dense_pyr_lk(const float* from, const float* to, int w, int h,
                          const fs_flow_params* params, float* vec, uint8_t* valid,
                          void* stream) {
    return guarded([&] {
        validate_flow_params(*params);
        if (w <= 0 || h <= 0) raise(FS_ERR_CONTRACT, "dense_pyr_lk: empty image");
        Stage st(stream);
        size_t n = (size_t)w * h;
        run_flow(st, st.in(from, n), st.in(to, n), w, h, *params, 1, vec, valid, nullptr, nullptr);
        st.finish();
    });
}

// flow.hpp:56-58 / src/flow.cpp:316-328
fs_status fs_bidirectional_flow(const float* overlapped_l, const float* overlapped_r, int w,
                                int h, int ch, const fs_flow_params* params, float* vec_ltor,
                                uint8_t* valid_ltor, float* vec_rtol, uint8_t* valid_rtol,
                                void* stream) {
    return guarded([&] {
        check_ch(ch);
        validate_flow_params(*params);
        if (w <= 0 || h <= 0) raise(FS_ERR_CONTRACT, "dense_pyr_lk: empty image");
        Stage st(stream);
        size_t n = (size_t)w * h;
        float* gl = st.tmp<float>(n);
        float* gr = st.tmp<float>(n);
        api::to_gray(st.in(overlapped_l, n * ch), (int)n, ch, gl, st.s);
        api::to_gray(st.in(overlapped_r, n * ch), (int)n, ch, gr, st.s);
        run_flow(st, gl, gr, w, h, *params, 2, vec_ltor, valid_ltor, vec_rtol, valid_rtol);
        st.finish();
    });
}

// flow.hpp:61 / src/flow.cpp:330-340
fs_status fs_flow_magnitude(const float* vec, int w, int h, float* out, void* stream) {
    return guarded([&] {
        size_t n = (size_t)w * h;
        Stage st(stream);
        if (n)
            api::magnitude(reinterpret_cast<const float2*>(st.in(vec, 2 * n)), n, st.out(out, n),
                           st.s);
        st.finish();
    });
}

// flow.hpp:65-66 / src/flow.cpp:342-355
fs_status fs_embed_flow(const float* vec, const uint8_t* valid, int w, int h, int offset_x,
                        int offset_y, int canvas_w, int canvas_h, float* out_vec,
                        uint8_t* out_valid, void* stream) {
    return guarded([&] {
        if (offset_x < 0 || offset_y < 0 || offset_x + w > canvas_w || offset_y + h > canvas_h)
            raise(FS_ERR_CONTRACT, "embed_flow: crop box does not fit inside the canvas");
        Stage st(stream);
        size_t n = (size_t)w * h, nc = (size_t)canvas_w * canvas_h;
        api::embed(reinterpret_cast<const float2*>(st.in(vec, 2 * n)), st.in(valid, n), w, h,
                   offset_x, offset_y, canvas_w, canvas_h,
                   reinterpret_cast<float2*>(st.out(out_vec, 2 * nc)), st.out(out_valid, nc), st.s);
        st.finish();
    });
}

// blend_field.hpp:32 / src/blend_field.cpp:51-86
fs_status fs_distance_transform(const uint8_t* mask, int w, int h, double* out, void* stream) {
    return guarded([&] {
        if (w <= 0 || h <= 0) raise(FS_ERR_CONTRACT, "distance_transform: empty canvas");
        check_edt_extent(w, h, "distance_transform");
        Stage st(stream);
        size_t n = (size_t)w * h;
        const uint8_t* dm = st.in(mask, n);
        auto* cnt = st.tmp<unsigned long long>(1);
        FS_CK(cudaMemsetAsync(cnt, 0, sizeof(unsigned long long), st.s));
        api::count_nonzero(dm, n, cnt, st.s);
        unsigned long long hc = 0;
        st.read(&hc, cnt, 1);
        if (hc == 0) raise(FS_ERR_EMPTY_REGION, "distance_transform: mask has no true pixel");
        int* dsq = st.tmp<int>(n);
        full_edt(st, PlaneMask{dm, w}, static_cast<const PlaneMask*>(nullptr), w, h, dsq, nullptr);
        api::sqrt_field(dsq, n, st.out(out, n), st.s);
        st.finish();
    });
}

// blend_field.hpp:34 / src/blend_field.cpp:88-130
fs_status fs_compute_blend(const uint8_t* label, const int64_t* counts, int w, int h, double* b,
                           void* stream) {
    return guarded([&] {
        check_dims(w, h);
        check_edt_extent(w, h, "compute_blend");
        int64_t c[4];
        read_counts(counts, c);
        Stage st(stream);
        size_t n = (size_t)w * h;
        if (n == 0) return;
        const uint8_t* dl = st.in(label, n);
        bool have1 = c[1] > 0, have2 = c[2] > 0;
        int *d1 = nullptr, *d2 = nullptr;
        if (have1 && have2 && c[3] > 0) {
            d1 = st.tmp<int>(n);
            d2 = st.tmp<int>(n);
            LabelMask m1{dl, w, 1}, m2{dl, w, 2};
            full_edt(st, m1, &m2, w, h, d1, d2);
        }
        api::blend_field(dl, n, have1, have2, d1, d2, st.out(b, n), st.s);
        st.finish();
    });
}

// blender.hpp:21-23 / src/blender.cpp:18-30
void fs_softmax_weights(double blend_l, double blend_r, double mag_rtol, double mag_ltor,
                        const fs_blend_params* params, double* sl, double* sr) {
    softmax_weights(blend_l, blend_r, mag_rtol, mag_ltor, params->k_softmax_sharpness,
                    params->k_flow_mag_coef, *sl, *sr);
}

// blender.hpp:30-33 / src/blender.cpp:43-100
fs_status fs_blend_pair(const float* l, const uint8_t* valid_l, const float* r,
                        const uint8_t* valid_r, int w, int h, int ch, const float* flow_ltor,
                        const float* flow_rtol, const double* blend, const uint8_t* label,
                        const fs_blend_params* params, float* out, uint8_t* out_valid,
                        void* stream) {
    return guarded([&] {
        validate_blend_params(*params);
        check_ch(ch);
        Stage st(stream);
        size_t n = (size_t)w * h;
        if (n == 0) return;
        const float* flr = st.in(flow_ltor, 2 * n);
        const float* frl = st.in(flow_rtol, 2 * n);
        auto* bad = st.tmp<unsigned long long>(1);
        FS_CK(cudaMemsetAsync(bad, 0, sizeof(unsigned long long), st.s));
        api::count_nonfinite(flr, 2 * n, bad, st.s);
        api::count_nonfinite(frl, 2 * n, bad, st.s);
        unsigned long long hb = 0;
        st.read(&hb, bad, 1);
        if (hb) raise(FS_ERR_CONTRACT, "blend_pair: non-finite flow");
        api::blend_pair(st.in(l, n * ch), st.in(valid_l, n), st.in(r, n * ch), st.in(valid_r, n), w,
                        h, ch, reinterpret_cast<const float2*>(flr),
                        reinterpret_cast<const float2*>(frl), st.in(blend, n), st.in(label, n),
                        params->k_softmax_sharpness, params->k_flow_mag_coef,
                        st.out(out, n * ch), st.out(out_valid, n), st.s);
        st.finish();
    });
}

// blender.hpp:36-37 / src/blender.cpp:102-135
fs_status fs_feather_blend(const float* l, const uint8_t* valid_l, const float* r,
                           const uint8_t* valid_r, int w, int h, int ch, const double* blend,
                           const uint8_t* label, float* out, uint8_t* out_valid, void* stream) {
    (void)valid_l;
    (void)valid_r;
    return guarded([&] {
        check_ch(ch);
        Stage st(stream);
        size_t n = (size_t)w * h;
        if (n == 0) return;
        api::feather(st.in(l, n * ch), st.in(r, n * ch), w, h, ch, st.in(blend, n),
                     st.in(label, n), st.out(out, n * ch), st.out(out_valid, n), st.s);
        st.finish();
    });
}

// blender.hpp:42-46 / src/blender.cpp:137-163
// pipeline.hpp:81-83 / src/pipeline.cpp:309-396
fs_status fs_misalignment_score(const float* l, const uint8_t* valid_l, const float* r,
                                const uint8_t* valid_r, int w, int h, int ch,
                                const uint8_t* label, const int64_t* counts, int patch_radius,
                                int stride, double* out, void* stream) {
    (void)valid_l;  // the reference reads only R's validity (src/pipeline.cpp:338)
    return guarded([&] {
        check_dims(w, h);
        check_ch(ch);
        int64_t c[4];
        read_counts(counts, c);
        if (c[3] == 0) raise(FS_ERR_CONTRACT, "misalignment_score: Area3 is empty");
        if (patch_radius < 1 || stride < 1)
            raise(FS_ERR_CONTRACT, "misalignment_score: patch_radius and stride must be >= 1");
        if (patch_radius > metrics::misalign_max_radius())
            raise(FS_ERR_UNSUPPORTED, "misalignment_score: patch_radius above the kernel's maximum");
        Stage st(stream);
        const size_t n = (size_t)w * h;
        const int ngx = w - 2 * patch_radius > 0 ? (w - 2 * patch_radius + stride - 1) / stride : 0;
        const int ngy = h - 2 * patch_radius > 0 ? (h - 2 * patch_radius + stride - 1) / stride : 0;
        int* res = st.tmp<int>(3 * (size_t)std::max(1, ngx * ngy));
        double* dout = st.tmp<double>(2);
        metrics::misalign(st.in(l, n * ch), st.in(r, n * ch), st.in(valid_r, n), st.in(label, n), w,
                          h, ch, patch_radius, stride, res, dout, st.s);
        double hout[2];
        st.read(hout, dout, 2);
        st.finish();
        if (hout[1] == 0.0) raise(FS_ERR_EMPTY_REGION, "misalignment_score: no textured patches");
        *out = hout[0];
    });
}

// pipeline.hpp:69-77 / src/pipeline.cpp:261-307
fs_status fs_estimate_translation(const float* a, const float* b, int w, int h, int ch,
                                  int max_shift, int* dx, int* dy, double* score, void* stream) {
    return guarded([&] {
        check_dims(w, h);
        if (ch != 1) raise(FS_ERR_CONTRACT, "estimate_translation: grayscale inputs required");
        if (max_shift > std::min(w, h) / 4)
            raise(FS_ERR_CONTRACT, "estimate_translation: max_shift too large for the image size");
        if (max_shift < 0) raise(FS_ERR_EMPTY_REGION, "estimate_translation: no texture");
        Stage st(stream);
        const size_t n = (size_t)w * h;
        double* ncc = st.tmp<double>((size_t)(2 * max_shift + 1) * (2 * max_shift + 1));
        double* dout = st.tmp<double>(4);
        metrics::translation(st.in(a, n), st.in(b, n), w, h, max_shift, ncc, dout, st.s);
        double hout[4];
        st.read(hout, dout, 4);
        st.finish();
        if (hout[0] == 0.0) raise(FS_ERR_EMPTY_REGION, "estimate_translation: no texture");
        *dx = (int)hout[1];
        *dy = (int)hout[2];
        *score = hout[3];
    });
}

fs_status fs_warp_constituents(const float* l, const uint8_t* valid_l, const float* r,
                               const uint8_t* valid_r, int w, int h, int ch,
                               const float* flow_ltor, const float* flow_rtol,
                               const double* blend, const uint8_t* label, float* out_l,
                               uint8_t* out_valid_l, float* out_r, uint8_t* out_valid_r,
                               void* stream) {
    return guarded([&] {
        check_ch(ch);
        Stage st(stream);
        size_t n = (size_t)w * h;
        if (n == 0) return;
        const float* dl = st.in(l, n * ch);
        const float* dr = st.in(r, n * ch);
        const uint8_t* dvl = st.in(valid_l, n);
        const uint8_t* dvr = st.in(valid_r, n);
        float* ol = st.out(out_l, n * ch);
        float* orr = st.out(out_r, n * ch);
        uint8_t* ovl = st.out(out_valid_l, n);
        uint8_t* ovr = st.out(out_valid_r, n);
        FS_CK(cudaMemcpyAsync(ol, dl, n * ch * sizeof(float), cudaMemcpyDeviceToDevice, st.s));
        FS_CK(cudaMemcpyAsync(orr, dr, n * ch * sizeof(float), cudaMemcpyDeviceToDevice, st.s));
        FS_CK(cudaMemcpyAsync(ovl, dvl, n, cudaMemcpyDeviceToDevice, st.s));
        FS_CK(cudaMemcpyAsync(ovr, dvr, n, cudaMemcpyDeviceToDevice, st.s));
        api::warp_constituents(dl, dvl, dr, dvr, w, h, ch,
                               reinterpret_cast<const float2*>(st.in(flow_ltor, 2 * n)),
                               reinterpret_cast<const float2*>(st.in(flow_rtol, 2 * n)),
                               st.in(blend, n), st.in(label, n), ol, ovl, orr, ovr, st.s);
        st.finish();
    });
}

// pipeline.hpp:63-67 / src/pipeline.cpp:140-212 (the fold; with stats, the
// report's seam metrics too)
fs_status fs_stitch_placed(int n, const float* const* images, const uint8_t* const* valids,
                           const int* dims, const int* offsets, int ch, int canvas_w,
                           int canvas_h, const fs_flow_params* flow, const fs_blend_params* blend,
                           float* out, uint8_t* out_valid, fs_pair_stats* stats, void* stream) {
    return guarded([&] {
        if (n < 2) raise(FS_ERR_CONTRACT, "stitch: at least two images required");
        validate_flow_params(*flow);
        validate_blend_params(*blend);
        check_ch(ch);
        check_edt_extent(canvas_w, canvas_h, "stitch");
        Stage st(stream);
        const size_t nc = (size_t)canvas_w * canvas_h;
        Canvas cv;
        cv.w = canvas_w;
        cv.h = canvas_h;
        cv.ch = ch;
        cv.rgb = st.tmp<float4>(nc);
        cv.valid = st.tmp<uint8_t>(nc);
        auto* cc = st.tmp<CanvasCount>(1);
        FS_CK(cudaMemsetAsync(cv.valid, 0, nc, st.s));
        init_count(cc, st.s);
        auto make_view = [&](int k) {
            int w = dims[2 * k], h = dims[2 * k + 1];
            int ox = offsets[2 * k], oy = offsets[2 * k + 1];
            if (ox < 0 || oy < 0 || ox + w > canvas_w || oy + h > canvas_h)
                raise(FS_ERR_LAYOUT, "place_on_canvas: image does not fit inside the canvas");
            size_t np = (size_t)w * h;
            ViewF4 v;
            v.rect = Rect{ox, oy, w, h};
            float4* px = st.tmp<float4>(np);
            uint8_t* vv = st.tmp<uint8_t>(np);
            if (np)
                api::import_view(st.in(images[k], np * ch),
                                 valids && valids[k] ? st.in(valids[k], np) : nullptr, np, ch, px,
                                 vv, st.s);
            v.px = px;
            v.valid = vv;
            return v;
        };
        ViewF4 v0 = make_view(0);
        if (v0.rect.w > 0 && v0.rect.h > 0) launch::place_view(cv, v0, cc, st.s);
        // union of the placed rectangles = a superset of the pano's valid bbox
        Rect pb = v0.rect;
        cudaEvent_t ev[4];
        for (auto& e : ev) FS_CK(cudaEventCreate(&e));
        std::unique_ptr<cudaEvent_t[], void (*)(cudaEvent_t*)> guard(ev, [](cudaEvent_t* e) {
            for (int q = 0; q < 4; ++q) cudaEventDestroy(e[q]);
        });
        double* magscratch = st.tmp<double>(257 * 2);
        for (int k = 1; k < n; ++k) {
            ViewF4 v = make_view(k);
            FoldWS<ViewF4> f;
            FoldStats* fst = st.tmp<FoldStats>(1);
            f.st = fst;
            const PanoPlane pano{cv.valid, cv.rgb, cv.w};
            init_stats(fst, st.s);
            if (v.rect.w > 0 && v.rect.h > 0) launch::partition(pano, v, fst, st.s);
            launch::snapshot_count(fst, cc, st.s);
            FoldStats hs;
            st.read(&hs, fst, 1);
            if (hs.cnt3 == 0)
                raise(FS_ERR_EMPTY_REGION,
                      "stitch: no overlap between the panorama and image #" + std::to_string(k));
            Rect box{hs.bx0, hs.by0, hs.bx1 - hs.bx0 + 1, hs.by1 - hs.by0 + 1};
            Arena a0;
            f.layout(a0, box, pb, v.rect, *flow);
            Arena a1;
            a1.base = static_cast<char*>(st.alloc(a0.off));
            f.layout(a1, box, pb, v.rect, *flow);
            FS_CK(cudaMemcpyAsync(f.st, fst, sizeof(FoldStats), cudaMemcpyDeviceToDevice, st.s));
            fold_enqueue_flow_edt(f, pano, pano, v, ch, *flow, st.s, ev[0], ev[1]);
            FoldStats hs2;
            st.read(&hs2, f.st, 1);
            if (hs2.edt_fail) {  // bounded domain not provably exact: redo on the full domain
                f.full_domain = true;
                f.replan_edt();
                fold_enqueue_flow_edt(f, pano, pano, v, ch, *flow, st.s, ev[0], ev[1]);
            }
            // seam metric of the raw pair, before the canvas is composed
            // (src/pipeline.cpp:184-187)
            double mis[2][2] = {{0, 0}, {0, 0}};
            int* mres = nullptr;
            double* mout = nullptr;
            if (stats) {
                mres = st.tmp<int>(3 * std::max<size_t>(1, metrics::fold_points(box, 8, 32)));
                mout = st.tmp<double>(4);
                metrics::misalign_fold(cv, v, box, nullptr, 8, 32, mres, mout, st.s);
                f.wgray = st.tmp<float2>((size_t)box.w * box.h);
                FS_CK(cudaMemsetAsync(f.wgray, 0xFF, sizeof(float2) * box.w * box.h, st.s));
            }
            FS_CK(cudaEventRecord(ev[2], st.s));
            fold_enqueue_blend(f, cv, v, cc, *blend, st.s);
            FS_CK(cudaEventRecord(ev[3], st.s));
            if (stats) {  // of the warped constituents (src/pipeline.cpp:192-199)
                metrics::misalign_fold(cv, v, box, f.wgray, 8, 32, mres, mout + 2, st.s);
                st.read(&mis[0][0], mout, 4);
            }
            if (stats) {
                api::mean_magnitude(f.fvec[0], (size_t)box.w * box.h, magscratch, st.s);
                api::mean_magnitude(f.fvec[1], (size_t)box.w * box.h, magscratch + 257, st.s);
                double m0 = 0, m1 = 0;
                st.read(&m0, magscratch, 1);
                st.read(&m1, magscratch + 257, 1);
                float tf = 0.f, tb = 0.f;
                FS_CK(cudaEventSynchronize(ev[3]));
                cudaEventElapsedTime(&tf, ev[0], ev[1]);
                cudaEventElapsedTime(&tb, ev[2], ev[3]);
                fs_pair_stats& ps = stats[k - 1];
                ps.overlap_pixels = (int64_t)hs.cnt3;
                ps.mean_flow_mag_ltor = m0;
                ps.mean_flow_mag_rtol = m1;
                ps.flow_seconds = tf * 1e-3;
                ps.blend_seconds = tb * 1e-3;
                ps.crop_box[0] = box.x0;
                ps.crop_box[1] = box.y0;
                ps.crop_box[2] = box.w;
                ps.crop_box[3] = box.h;
                ps.misalignment_present = (mis[0][1] > 0 ? 1 : 0) | (mis[1][1] > 0 ? 2 : 0);
                ps.misalignment_before = mis[0][1] > 0 ? mis[0][0] : 0.0;
                ps.misalignment_after = mis[1][1] > 0 ? mis[1][0] : 0.0;
            }
            // grow the pano bbox by the placed rectangle
            int x0 = std::min(pb.x0, v.rect.x0), y0 = std::min(pb.y0, v.rect.y0);
            int x1 = std::max(pb.x1(), v.rect.x1()), y1 = std::max(pb.y1(), v.rect.y1());
            pb = Rect{x0, y0, x1 - x0, y1 - y0};
        }
        launch::export_float(cv, st.out(out, nc * ch), st.out(out_valid, nc), st.s);
        st.finish();
    });
}

}  // extern "C"
