// TEST INFRASTRUCTURE (oracle) — not product code.
//
// extern "C" shims over the UNMODIFIED reference library (compiled from
// /root/reference/proj/src by oracle/Makefile into oracle/_ref/libfsref.so).
// Each fsref_* has the parameter list of the matching fso_* in fs_oracle.h,
// converts plain buffers to the reference value types, calls the reference
// function named in its comment and copies the result back.  Exceptions map to
// the FSO_* status codes (proj/include/flowstitch/errors.hpp:10-37).
#include <chrono>
#include <cmath>
#include <cstring>
#include <vector>

#include "flowstitch/blend_field.hpp"
#include "flowstitch/blender.hpp"
#include "flowstitch/errors.hpp"
#include "flowstitch/flow.hpp"
#include "flowstitch/image.hpp"
#include "flowstitch/parallel.hpp"
#include "flowstitch/pipeline.hpp"
#include "fs_oracle.h"

using namespace flowstitch;

namespace {

ImageBuf make_image(const float* data, const uint8_t* valid, int w, int h, int ch) {
    ImageBuf img(w, h, ch);
    std::memcpy(img.data().data(), data, sizeof(float) * static_cast<size_t>(w) * h * ch);
    if (valid)
        for (int j = 0; j < h; ++j)
            for (int i = 0; i < w; ++i) img.set_valid(i, j, valid[static_cast<size_t>(j) * w + i] != 0);
    return img;
}

void export_image(const ImageBuf& img, float* data, uint8_t* valid) {
    std::memcpy(data, img.data().data(), sizeof(float) * img.data().size());
    if (valid)
        for (int j = 0; j < img.height(); ++j)
            for (int i = 0; i < img.width(); ++i)
                valid[static_cast<size_t>(j) * img.width() + i] = img.valid(i, j) ? 1 : 0;
}

Mask make_mask(const uint8_t* m, int w, int h) {
    Mask mask(w, h);
    std::memcpy(mask.v.data(), m, static_cast<size_t>(w) * h);
    return mask;
}

RegionPartition make_partition(const uint8_t* label, const int64_t* counts, int w, int h) {
    RegionPartition p;
    p.width = w;
    p.height = h;
    p.label.resize(static_cast<size_t>(w) * h);
    for (size_t k = 0; k < p.label.size(); ++k) p.label[k] = static_cast<Region>(label[k]);
    for (int r = 0; r < 4; ++r) p.counts[r] = counts[r];
    return p;
}

FlowField make_flow(const float* vec, int w, int h) {
    FlowField f(w, h);
    std::memcpy(f.vec.data(), vec, sizeof(float) * 2 * static_cast<size_t>(w) * h);
    return f;
}

FlowParams flow_params(int levels, int radius, int iters, double eps, int smoothing) {
    FlowParams p;
    p.levels = levels;
    p.window_radius = radius;
    p.iterations_per_level = iters;
    p.min_eigen_eps = eps;
    p.smoothing_passes = smoothing;
    return p;
}

template <class F>
int guarded(F&& fn) {
    try {
        fn();
        return FSO_OK;
    } catch (const EmptyRegionError&) {
        return FSO_EMPTY;
    } catch (const LayoutError&) {
        return FSO_LAYOUT;
    } catch (const ContractError&) {
        return FSO_CONTRACT;
    }
}

StitchReport& last_report() {
    static StitchReport rep;
    return rep;
}

void export_flow(const FlowField& f, float* vec, uint8_t* valid) {
    std::memcpy(vec, f.vec.data(), sizeof(float) * f.vec.size());
    std::memcpy(valid, f.valid.data(), f.valid.size());
}

} // namespace

extern "C" {

void fsref_set_threads(int n) { set_thread_count(n); }
int fsref_resolved_threads() { return resolved_thread_count(); }

// proj/src/image.cpp:70-83
int fsref_to_gray(const float* img, int w, int h, int ch, float* out) {
    return guarded([&] {
        ImageBuf g = to_gray(make_image(img, nullptr, w, h, ch));
        std::memcpy(out, g.data().data(), sizeof(float) * g.data().size());
    });
}

// proj/src/image.cpp:85-113
void fsref_bilinear_sample(const float* img, const uint8_t* valid, int w, int h, int ch, double x,
                           double y, float* out) {
    bilinear_sample(make_image(img, valid, w, h, ch), x, y, out);
}

// proj/src/image.cpp:115-132
int fsref_compute_partition(const uint8_t* ml, const uint8_t* mr, int w, int h, uint8_t* label,
                            int64_t* counts) {
    return guarded([&] {
        RegionPartition p = compute_partition(make_mask(ml, w, h), make_mask(mr, w, h));
        for (size_t k = 0; k < p.label.size(); ++k) label[k] = static_cast<uint8_t>(p.label[k]);
        for (int r = 0; r < 4; ++r) counts[r] = p.counts[r];
    });
}

// proj/src/image.cpp:134-162
int fsref_crop_overlap(const float* img, const uint8_t* valid, int w, int h, int ch,
                       const uint8_t* label, const int64_t* counts, float* out, uint8_t* out_valid,
                       int* box) {
    return guarded([&] {
        CropResult c = crop_overlap(make_image(img, valid, w, h, ch),
                                    make_partition(label, counts, w, h));
        box[0] = c.offset_x;
        box[1] = c.offset_y;
        box[2] = c.image.width();
        box[3] = c.image.height();
        if (out) export_image(c.image, out, out_valid);
    });
}

// proj/src/image.cpp:164-177
int fsref_place_on_canvas(const float* img, const uint8_t* valid, int w, int h, int ch, int ox,
                          int oy, int cw, int chh, float* out, uint8_t* out_valid) {
    return guarded([&] {
        export_image(place_on_canvas(make_image(img, valid, w, h, ch), ox, oy, cw, chh), out,
                     out_valid);
    });
}

// proj/src/flow.cpp:174-192; returns the depth (or -status on error)
int fsref_build_pyramid(const float* img, int w, int h, int levels, float* out) {
    int depth = 0;
    int st = guarded([&] {
        auto pyr = build_pyramid(make_image(img, nullptr, w, h, 1), levels);
        size_t off = 0;
        for (const auto& lvl : pyr) {
            std::memcpy(out + off, lvl.data().data(), sizeof(float) * lvl.data().size());
            off += lvl.data().size();
        }
        depth = static_cast<int>(pyr.size());
    });
    return st == FSO_OK ? depth : -st;
}

// proj/src/flow.cpp:194-314
int fsref_dense_pyr_lk(const float* from, const float* to, int w, int h, int levels, int radius,
                       int iters, double eps, int smoothing, float* vec, uint8_t* valid) {
    return guarded([&] {
        FlowField f = dense_pyr_lk(make_image(from, nullptr, w, h, 1),
                                   make_image(to, nullptr, w, h, 1),
                                   flow_params(levels, radius, iters, eps, smoothing));
        export_flow(f, vec, valid);
    });
}

// proj/src/flow.cpp:316-328
int fsref_bidirectional_flow(const float* l, const float* r, int w, int h, int ch, int levels,
                             int radius, int iters, double eps, int smoothing, float* vec_lr,
                             uint8_t* valid_lr, float* vec_rl, uint8_t* valid_rl) {
    return guarded([&] {
        auto [lr, rl] = bidirectional_flow(make_image(l, nullptr, w, h, ch),
                                           make_image(r, nullptr, w, h, ch),
                                           flow_params(levels, radius, iters, eps, smoothing));
        export_flow(lr, vec_lr, valid_lr);
        export_flow(rl, vec_rl, valid_rl);
    });
}

// proj/src/flow.cpp:342-355
int fsref_embed_flow(const float* vec, const uint8_t* valid, int w, int h, int ox, int oy, int cw,
                     int chh, float* out_vec, uint8_t* out_valid) {
    return guarded([&] {
        FlowField f = make_flow(vec, w, h);
        std::memcpy(f.valid.data(), valid, f.valid.size());
        export_flow(embed_flow(f, ox, oy, cw, chh), out_vec, out_valid);
    });
}

// proj/src/flow.cpp:330-340
void fsref_flow_magnitude(const float* vec, int w, int h, float* out) {
    auto m = flow_magnitude(make_flow(vec, w, h));
    std::memcpy(out, m.data(), sizeof(float) * m.size());
}

// proj/src/blend_field.cpp:51-86
int fsref_distance_transform(const uint8_t* mask, int w, int h, double* out) {
    return guarded([&] {
        DistanceField d = distance_transform(make_mask(mask, w, h));
        std::memcpy(out, d.d.data(), sizeof(double) * d.d.size());
    });
}

// proj/src/blend_field.cpp:88-130
int fsref_compute_blend(const uint8_t* label, const int64_t* counts, int w, int h, double* b) {
    return guarded([&] {
        BlendField f = compute_blend(make_partition(label, counts, w, h));
        std::memcpy(b, f.b.data(), sizeof(double) * f.b.size());
    });
}

// proj/src/blender.cpp:18-30
void fsref_softmax_weights(double bl, double br, double mrl, double mlr, double k, double coef,
                           double* out2) {
    BlendParams p;
    p.k_softmax_sharpness = k;
    p.k_flow_mag_coef = coef;
    auto [sl, sr] = softmax_weights(bl, br, mrl, mlr, p);
    out2[0] = sl;
    out2[1] = sr;
}

// proj/src/blender.cpp:43-100
int fsref_blend_pair(const float* l, const uint8_t* vl, const float* r, const uint8_t* vr, int w,
                     int h, int ch, const float* flow_lr, const float* flow_rl, const double* b,
                     const uint8_t* label, double k, double coef, float* out, uint8_t* out_valid) {
    return guarded([&] {
        int64_t counts[4] = {0, 0, 0, 0};
        for (size_t q = 0; q < static_cast<size_t>(w) * h; ++q) ++counts[label[q]];
        BlendField bf;
        bf.width = w;
        bf.height = h;
        bf.b.assign(b, b + static_cast<size_t>(w) * h);
        BlendParams p;
        p.k_softmax_sharpness = k;
        p.k_flow_mag_coef = coef;
        ImageBuf f = blend_pair(make_image(l, vl, w, h, ch), make_image(r, vr, w, h, ch),
                                make_flow(flow_lr, w, h), make_flow(flow_rl, w, h), bf,
                                make_partition(label, counts, w, h), p);
        export_image(f, out, out_valid);
    });
}

// proj/src/blender.cpp:102-135
int fsref_feather_blend(const float* l, const float* r, int w, int h, int ch, const double* b,
                        const uint8_t* label, float* out, uint8_t* out_valid) {
    return guarded([&] {
        int64_t counts[4] = {0, 0, 0, 0};
        for (size_t q = 0; q < static_cast<size_t>(w) * h; ++q) ++counts[label[q]];
        BlendField bf;
        bf.width = w;
        bf.height = h;
        bf.b.assign(b, b + static_cast<size_t>(w) * h);
        ImageBuf f = feather_blend(make_image(l, nullptr, w, h, ch), make_image(r, nullptr, w, h, ch),
                                   bf, make_partition(label, counts, w, h));
        export_image(f, out, out_valid);
    });
}

// proj/src/blender.cpp:137-163
int fsref_warp_constituents(const float* l, const uint8_t* vl, const float* r, const uint8_t* vr,
                            int w, int h, int ch, const float* flow_lr, const float* flow_rl,
                            const double* b, const uint8_t* label, float* out_l, uint8_t* out_vl,
                            float* out_r, uint8_t* out_vr) {
    return guarded([&] {
        int64_t counts[4] = {0, 0, 0, 0};
        for (size_t q = 0; q < static_cast<size_t>(w) * h; ++q) ++counts[label[q]];
        BlendField bf;
        bf.width = w;
        bf.height = h;
        bf.b.assign(b, b + static_cast<size_t>(w) * h);
        auto pr = warp_constituents(make_image(l, vl, w, h, ch), make_image(r, vr, w, h, ch),
                                    make_flow(flow_lr, w, h), make_flow(flow_rl, w, h), bf,
                                    make_partition(label, counts, w, h));
        export_image(pr.first, out_l, out_vl);
        export_image(pr.second, out_r, out_vr);
    });
}

namespace {

using Clock = std::chrono::steady_clock;
double secs(Clock::time_point a, Clock::time_point b) {
    return std::chrono::duration<double>(b - a).count();
}

std::vector<PlacedImage> make_placed(int n, const float* const* imgs, const uint8_t* const* valids,
                                     const int* dims, const int* offsets, int ch) {
    std::vector<PlacedImage> placed(n);
    for (int k = 0; k < n; ++k) {
        placed[k].image = make_image(imgs[k], valids ? valids[k] : nullptr, dims[2 * k],
                                     dims[2 * k + 1], ch);
        placed[k].offset_x = offsets[2 * k];
        placed[k].offset_y = offsets[2 * k + 1];
    }
    return placed;
}

} // namespace

// The fold of proj/src/pipeline.cpp:150-204, calling the reference functions
// in the same order, minus misalignment_score / warp_constituents (:184-187,
// :194-199: metrics that never write the panorama).  `timing` (optional,
// 5 doubles): prep (place/partition/crop), flow, embed, blend field, blend.
// `fold_cb` (optional) receives every fold's crop flows (the reference's own
// bidirectional_flow output, proj/src/pipeline.cpp:171-172) and crop box;
// the time it takes is excluded from `timing`.  timing[5] (when timing is
// given) = seconds of the whole fold, the callbacks excluded.
typedef void (*fsref_fold_cb)(int k, int ox, int oy, int w, int h, const float* lr,
                              const uint8_t* lr_valid, const float* rl, const uint8_t* rl_valid,
                              void* ctx);
int fsref_stitch_placed_flows(int n, const float* const* imgs, const uint8_t* const* valids,
                              const int* dims, const int* offsets, int ch, int cw, int chh,
                              int levels, int radius, int iters, double eps, int smoothing,
                              double k, double coef, float* out, uint8_t* out_valid,
                              double* timing, fsref_fold_cb fold_cb, void* ctx) {
    auto t_start = Clock::now();
    double cb_s = 0.0;
    std::vector<PlacedImage> placed = make_placed(n, imgs, valids, dims, offsets, ch);
    double t[5] = {0, 0, 0, 0, 0};
    int st = guarded([&] {
        FlowParams fp = flow_params(levels, radius, iters, eps, smoothing);
        BlendParams bp;
        bp.k_softmax_sharpness = k;
        bp.k_flow_mag_coef = coef;
        if (placed.size() < 2) throw ContractError("stitch: at least two images required");
        fp.validate();
        bp.validate();
        auto t0 = Clock::now();
        ImageBuf pano = place_on_canvas(placed[0].image, placed[0].offset_x, placed[0].offset_y,
                                        cw, chh);
        t[0] += secs(t0, Clock::now());
        for (size_t kk = 1; kk < placed.size(); ++kk) {
            auto a = Clock::now();
            ImageBuf next = place_on_canvas(placed[kk].image, placed[kk].offset_x,
                                            placed[kk].offset_y, cw, chh);
            if (pano.channels() != next.channels())
                throw ContractError("stitch: mixed grayscale and color inputs");
            RegionPartition part = compute_partition(pano.valid_mask(), next.valid_mask());
            if (part.count(Region::Area3) == 0)
                throw EmptyRegionError("stitch: no overlap");
            CropResult crop_l = crop_overlap(pano, part);
            CropResult crop_r = crop_overlap(next, part);
            auto b = Clock::now();
            auto [lr_c, rl_c] = bidirectional_flow(crop_l.image, crop_r.image, fp);
            auto c = Clock::now();
            if (fold_cb) {
                fold_cb(static_cast<int>(kk), crop_l.offset_x, crop_l.offset_y, lr_c.width,
                        lr_c.height, lr_c.vec.data(), lr_c.valid.data(), rl_c.vec.data(),
                        rl_c.valid.data(), ctx);
                auto c2 = Clock::now();
                cb_s += secs(c, c2);
                c = c2;
            }
            FlowField lr = embed_flow(lr_c, crop_l.offset_x, crop_l.offset_y, cw, chh);
            FlowField rl = embed_flow(rl_c, crop_l.offset_x, crop_l.offset_y, cw, chh);
            auto d = Clock::now();
            BlendField blend = compute_blend(part);
            auto e = Clock::now();
            ImageBuf blended = blend_pair(pano, next, lr, rl, blend, part, bp);
            for (int j = 0; j < chh; ++j)
                for (int i = 0; i < cw; ++i) blended.set_valid(i, j, pano.valid(i, j) || next.valid(i, j));
            pano = std::move(blended);
            auto f = Clock::now();
            t[0] += secs(a, b);
            t[1] += secs(b, c);
            t[2] += secs(c, d);
            t[3] += secs(d, e);
            t[4] += secs(e, f);
        }
        export_image(pano, out, out_valid);
    });
    if (timing) {
        for (int q = 0; q < 5; ++q) timing[q] = t[q];
        timing[5] = secs(t_start, Clock::now()) - cb_s;
    }
    return st;
}

int fsref_stitch_placed_timed(int n, const float* const* imgs, const uint8_t* const* valids,
                              const int* dims, const int* offsets, int ch, int cw, int chh,
                              int levels, int radius, int iters, double eps, int smoothing,
                              double k, double coef, float* out, uint8_t* out_valid,
                              double* timing) {
    double t6[6];
    int st = fsref_stitch_placed_flows(n, imgs, valids, dims, offsets, ch, cw, chh, levels, radius,
                                       iters, eps, smoothing, k, coef, out, out_valid, t6, nullptr,
                                       nullptr);
    if (timing)
        for (int q = 0; q < 5; ++q) timing[q] = t6[q];
    return st;
}

int fsref_stitch_placed(int n, const float* const* imgs, const uint8_t* const* valids,
                        const int* dims, const int* offsets, int ch, int cw, int chh, int levels,
                        int radius, int iters, double eps, int smoothing, double k, double coef,
                        float* out, uint8_t* out_valid) {
    return fsref_stitch_placed_timed(n, imgs, valids, dims, offsets, ch, cw, chh, levels, radius,
                                     iters, eps, smoothing, k, coef, out, out_valid, nullptr);
}

// proj/src/pipeline.cpp:309-396
int fsref_misalignment_score(const float* l, const uint8_t* l_valid, const float* r,
                             const uint8_t* r_valid, int w, int h, int ch, const uint8_t* label,
                             const int64_t* counts, int patch_radius, int stride, double* out) {
    return guarded([&] {
        *out = misalignment_score(make_image(l, l_valid, w, h, ch), make_image(r, r_valid, w, h, ch),
                                  make_partition(label, counts, w, h), patch_radius, stride);
    });
}

// proj/src/pipeline.cpp:261-307
int fsref_estimate_translation(const float* a, const float* b, int w, int h, int ch, int max_shift,
                               int* dx, int* dy, double* score) {
    return guarded([&] {
        TranslationEstimate t =
            estimate_translation(make_image(a, nullptr, w, h, ch), make_image(b, nullptr, w, h, ch),
                                 max_shift);
        *dx = t.dx;
        *dy = t.dy;
        *score = t.score;
    });
}

// The reference's own stitch_placed (proj/src/pipeline.cpp:140-212), metrics
// included; used to pin that the metric-free fold above yields the same canvas.
int fsref_stitch_placed_full(int n, const float* const* imgs, const uint8_t* const* valids,
                             const int* dims, const int* offsets, int ch, int cw, int chh,
                             int levels, int radius, int iters, double eps, int smoothing,
                             double k, double coef, float* out, uint8_t* out_valid) {
    return guarded([&] {
        BlendParams bp;
        bp.k_softmax_sharpness = k;
        bp.k_flow_mag_coef = coef;
        auto [pano, rep] = stitch_placed(make_placed(n, imgs, valids, dims, offsets, ch), cw, chh,
                                         flow_params(levels, radius, iters, eps, smoothing), bp);
        export_image(pano, out, out_valid);
        last_report() = rep;
    });
}

// The seam metrics of the last fsref_stitch_placed_full report: per pair
// (misalignment_before, misalignment_after), NaN where the optional is empty.
int fsref_last_report_misalignment(double* out, int max_pairs) {
    const auto& pairs = last_report().pairs;
    int n = 0;
    for (const auto& p : pairs) {
        if (n == max_pairs) break;
        out[2 * n] = p.misalignment_before ? *p.misalignment_before : NAN;
        out[2 * n + 1] = p.misalignment_after ? *p.misalignment_after : NAN;
        ++n;
    }
    return n;
}

} // extern "C"
