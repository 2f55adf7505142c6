// Drop-in C++ implementation of the reference's flow+blend API
// (namespace flowstitch, /root/reference/proj/include/flowstitch/
// {image,flow,blend_field,blender,parallel}.hpp) on top of the B200 C-ABI
// (include/fs_b200.h).  Compiled against the user's own copy of those headers,
// it replaces the reference's image.cpp / flow.cpp / blend_field.cpp /
// blender.cpp / parallel.cpp: every per-pixel computation runs in the sm_100a
// kernels; this file only converts value types, validates exactly like the
// reference (same exception types and messages) and maps C-ABI status codes
// back to exceptions.  The reference's pipeline.cpp links unchanged on top
// (its stitch_placed then drives the GPU functions fold by fold); the
// device-resident fold is flowstitch::b200::stitch_placed (pipeline_b200.cpp).
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <functional>
#include <thread>
#include <vector>

#include "flowstitch/blend_field.hpp"
#include "flowstitch/blender.hpp"
#include "flowstitch/errors.hpp"
#include "flowstitch/flow.hpp"
#include "flowstitch/image.hpp"
#include "flowstitch/parallel.hpp"
#include "fs_b200.h"
#include "png_io.hpp"

namespace flowstitch {

namespace {

// C-ABI status -> the reference's exception types (errors.hpp:10-37)
void check(fs_status st) {
    if (st == FS_OK) return;
    std::string msg = fs_last_error();
    switch (st) {
        case FS_ERR_CONTRACT:
        case FS_ERR_UNSUPPORTED: throw ContractError(msg);
        case FS_ERR_EMPTY_REGION: throw EmptyRegionError(msg);
        case FS_ERR_LAYOUT: throw LayoutError(msg);
        case FS_ERR_IO: throw IoError(msg);
        case FS_ERR_FORMAT: throw FormatError(msg);
        default: throw std::runtime_error("flowstitch-b200: " + msg);
    }
}

std::vector<uint8_t> valid_bytes(const ImageBuf& img) {
    std::vector<uint8_t> v(static_cast<size_t>(img.width()) * img.height());
    for (int j = 0; j < img.height(); ++j)
        for (int i = 0; i < img.width(); ++i)
            v[static_cast<size_t>(j) * img.width() + i] = img.valid(i, j) ? 1 : 0;
    return v;
}

void set_valid_bytes(ImageBuf& img, const std::vector<uint8_t>& v) {
    for (int j = 0; j < img.height(); ++j)
        for (int i = 0; i < img.width(); ++i)
            img.set_valid(i, j, v[static_cast<size_t>(j) * img.width() + i] != 0);
}

fs_flow_params to_c(const FlowParams& p) {
    return fs_flow_params{p.levels, p.window_radius, p.iterations_per_level, p.min_eigen_eps,
                          p.smoothing_passes};
}
fs_blend_params to_c(const BlendParams& p) {
    return fs_blend_params{p.k_softmax_sharpness, p.k_flow_mag_coef};
}

std::vector<uint8_t> labels_of(const RegionPartition& p) {
    std::vector<uint8_t> l(p.label.size());
    for (size_t k = 0; k < l.size(); ++k) l[k] = static_cast<uint8_t>(p.label[k]);
    return l;
}

}  // namespace

// ---------------------------------------------------------------- imagecore
ImageBuf::ImageBuf(int width, int height, int channels, float fill, bool valid)
    : width_(width), height_(height), channels_(channels),
      data_(static_cast<size_t>(width < 0 ? 0 : width) * (height < 0 ? 0 : height) *
                (channels < 0 ? 0 : channels),
            fill),
      valid_(static_cast<size_t>(width < 0 ? 0 : width) * (height < 0 ? 0 : height),
             valid ? 1 : 0) {
    if (width < 0 || height < 0 || (channels != 1 && channels != 3))
        throw ContractError("ImageBuf: channels must be 1 or 3");
}

Mask ImageBuf::valid_mask() const {
    Mask m(width_, height_);
    m.v = valid_;
    return m;
}

// Host image I/O on the PNG codec of png_codec.cpp.
// u8 -> float as load_image does it (src/image.cpp:27-43): value * (1.0f /
// 255.0f) in float, 1 channel for gray files, 3 otherwise, valid = alpha >= 128
// when the file has alpha.
ImageBuf load_image(const std::string& path) {
    detail::RawPng raw = detail::read_png(path);
    const int oc = raw.channels == 1 ? 1 : 3;
    ImageBuf img(raw.width, raw.height, oc);
    const float scale = 1.0f / 255.0f;
    const size_t n = static_cast<size_t>(raw.width) * raw.height;
    std::vector<float>& d = img.data();
    for (size_t k = 0; k < n; ++k) {
        const uint8_t* px = raw.bytes.data() + k * raw.channels;
        for (int c = 0; c < oc; ++c) d[k * oc + c] = px[c] * scale;
    }
    if (raw.channels == 4) {
        std::vector<uint8_t> v(n);
        for (size_t k = 0; k < n; ++k) v[k] = raw.bytes[k * 4 + 3] >= 128;
        set_valid_bytes(img, v);
    }
    return img;
}
// float -> u8 as save_image does it (src/image.cpp:45-68): alpha only when a
// pixel is invalid, lround(clamp(v, 0, 1) * 255.0f) (the product in float),
// gray replicated into RGB when alpha is added.
void save_image(const ImageBuf& img, const std::string& path) {
    if (img.empty()) throw ContractError("save_image: empty image");
    const std::vector<uint8_t> valid = valid_bytes(img);
    bool any_invalid = false;
    for (uint8_t v : valid) any_invalid |= v == 0;
    const int oc = img.channels() == 1 ? (any_invalid ? 4 : 1) : (any_invalid ? 4 : 3);
    const size_t n = static_cast<size_t>(img.width()) * img.height();
    std::vector<uint8_t> bytes(n * oc);
    const std::vector<float>& d = img.data();
    const int ic = img.channels();
    for (size_t k = 0; k < n; ++k) {
        uint8_t* px = bytes.data() + k * oc;
        for (int c = 0; c < std::min(oc, 3); ++c) {
            const float v = std::clamp(d[k * ic + std::min(c, ic - 1)], 0.0f, 1.0f);
            px[c] = static_cast<uint8_t>(std::lround(v * 255.0f));
        }
        if (oc == 4) px[3] = valid[k] ? 255 : 0;
    }
    detail::write_png(path, img.width(), img.height(), oc, bytes);
}

ImageBuf to_gray(const ImageBuf& img) {  // image.hpp:94
    if (img.channels() == 1) return img;
    ImageBuf g(img.width(), img.height(), 1);
    check(fs_to_gray(img.data().data(), img.width(), img.height(), img.channels(),
                     g.data().data(), nullptr));
    set_valid_bytes(g, valid_bytes(img));
    return g;
}

int bilinear_sample(const ImageBuf& img, double x, double y, float* out) {  // image.hpp:98
    const double xy[2] = {x, y};
    std::vector<uint8_t> v = valid_bytes(img);
    check(fs_bilinear_sample(img.data().data(), v.data(), img.width(), img.height(),
                             img.channels(), xy, 1, out, nullptr));
    return img.channels();
}

RegionPartition compute_partition(const Mask& maskL, const Mask& maskR) {  // image.hpp:100
    if (maskL.width != maskR.width || maskL.height != maskR.height)
        throw ContractError("compute_partition: mask dimensions differ");
    RegionPartition p;
    p.width = maskL.width;
    p.height = maskL.height;
    std::vector<uint8_t> label(static_cast<size_t>(p.width) * p.height);
    int64_t counts[4] = {0, 0, 0, 0};
    check(fs_compute_partition(maskL.v.data(), maskR.v.data(), p.width, p.height, label.data(),
                               counts, nullptr));
    p.label.resize(label.size());
    for (size_t k = 0; k < label.size(); ++k) p.label[k] = static_cast<Region>(label[k]);
    for (int r = 0; r < 4; ++r) p.counts[r] = counts[r];
    return p;
}

CropResult crop_overlap(const ImageBuf& img, const RegionPartition& partition) {  // image.hpp:103
    if (img.width() != partition.width || img.height() != partition.height)
        throw ContractError("crop_overlap: image and partition dimensions differ");
    if (partition.count(Region::Area3) == 0)
        throw EmptyRegionError("crop_overlap: no overlap (Area3 is empty)");
    std::vector<uint8_t> label = labels_of(partition), v = valid_bytes(img);
    int64_t counts[4];
    for (int r = 0; r < 4; ++r) counts[r] = partition.counts[r];
    int box[4];
    check(fs_crop_overlap(img.data().data(), v.data(), img.width(), img.height(), img.channels(),
                          label.data(), counts, nullptr, nullptr, box, nullptr));
    CropResult out;
    out.offset_x = box[0];
    out.offset_y = box[1];
    out.image = ImageBuf(box[2], box[3], img.channels());
    std::vector<uint8_t> ov(static_cast<size_t>(box[2]) * box[3]);
    check(fs_crop_overlap(img.data().data(), v.data(), img.width(), img.height(), img.channels(),
                          label.data(), counts, out.image.data().data(), ov.data(), box, nullptr));
    set_valid_bytes(out.image, ov);
    return out;
}

ImageBuf place_on_canvas(const ImageBuf& img, int offset_x, int offset_y, int canvas_width,
                         int canvas_height) {  // image.hpp:107-108
    if (offset_x < 0 || offset_y < 0 || offset_x + img.width() > canvas_width ||
        offset_y + img.height() > canvas_height)
        throw LayoutError("place_on_canvas: image does not fit inside the canvas");
    ImageBuf canvas(canvas_width, canvas_height, img.channels(), 0.0f, false);
    std::vector<uint8_t> v = valid_bytes(img), cv(static_cast<size_t>(canvas_width) * canvas_height);
    check(fs_place_on_canvas(img.data().data(), v.data(), img.width(), img.height(),
                             img.channels(), offset_x, offset_y, canvas_width, canvas_height,
                             canvas.data().data(), cv.data(), nullptr));
    set_valid_bytes(canvas, cv);
    return canvas;
}

// ---------------------------------------------------------------- optflow
void FlowParams::validate() const {  // src/flow.cpp:15-21 (same messages)
    if (levels < 1) throw ContractError("FlowParams: levels must be >= 1");
    if (window_radius < 1) throw ContractError("FlowParams: window_radius must be >= 1");
    if (iterations_per_level < 1) throw ContractError("FlowParams: iterations_per_level must be >= 1");
    if (!(min_eigen_eps > 0.0)) throw ContractError("FlowParams: min_eigen_eps must be > 0");
    if (smoothing_passes < 0) throw ContractError("FlowParams: smoothing_passes must be >= 0");
}

std::vector<ImageBuf> build_pyramid(const ImageBuf& img, int levels) {  // flow.hpp:48
    if (img.channels() != 1) throw ContractError("build_pyramid: grayscale input required");
    if (levels < 1) throw ContractError("build_pyramid: levels must be >= 1");
    int depth = fs_pyramid_depth(img.width(), img.height(), levels);
    size_t total = 0;
    std::vector<std::pair<int, int>> dims;
    int w = img.width(), h = img.height();
    for (int l = 0; l < depth; ++l) {
        dims.push_back({w, h});
        total += static_cast<size_t>(w) * h;
        w = std::max(1, w / 2);
        h = std::max(1, h / 2);
    }
    std::vector<float> all(total);
    int d = 0;
    check(fs_build_pyramid(img.data().data(), img.width(), img.height(), levels, all.data(), &d,
                           nullptr));
    std::vector<ImageBuf> pyr;
    size_t off = 0;
    for (int l = 0; l < depth; ++l) {
        ImageBuf lv(dims[l].first, dims[l].second, 1);
        std::memcpy(lv.data().data(), all.data() + off, sizeof(float) * lv.data().size());
        off += lv.data().size();
        pyr.push_back(std::move(lv));
    }
    pyr[0] = img;  // level 0 is the input itself (src/flow.cpp:189)
    return pyr;
}

FlowField dense_pyr_lk(const ImageBuf& from, const ImageBuf& to, const FlowParams& params) {
    params.validate();
    if (from.width() != to.width() || from.height() != to.height())
        throw ContractError("dense_pyr_lk: dimension mismatch");
    if (from.channels() != 1 || to.channels() != 1)
        throw ContractError("dense_pyr_lk: grayscale inputs required");
    FlowField out(from.width(), from.height());
    fs_flow_params p = to_c(params);
    check(fs_dense_pyr_lk(from.data().data(), to.data().data(), from.width(), from.height(), &p,
                          out.vec.data(), out.valid.data(), nullptr));
    return out;
}

std::pair<FlowField, FlowField> bidirectional_flow(const ImageBuf& overlappedL,
                                                   const ImageBuf& overlappedR,
                                                   const FlowParams& params) {
    if (overlappedL.width() != overlappedR.width() ||
        overlappedL.height() != overlappedR.height())
        throw ContractError("bidirectional_flow: dimension mismatch");
    params.validate();
    if (overlappedL.channels() != overlappedR.channels())
        throw ContractError("dense_pyr_lk: grayscale inputs required");
    const int w = overlappedL.width(), h = overlappedL.height();
    FlowField lr(w, h), rl(w, h);
    fs_flow_params p = to_c(params);
    check(fs_bidirectional_flow(overlappedL.data().data(), overlappedR.data().data(), w, h,
                                overlappedL.channels(), &p, lr.vec.data(), lr.valid.data(),
                                rl.vec.data(), rl.valid.data(), nullptr));
    return {std::move(lr), std::move(rl)};
}

std::vector<float> flow_magnitude(const FlowField& flow) {  // flow.hpp:61
    std::vector<float> mag(static_cast<size_t>(flow.width) * flow.height);
    if (!mag.empty())
        check(fs_flow_magnitude(flow.vec.data(), flow.width, flow.height, mag.data(), nullptr));
    return mag;
}

FlowField embed_flow(const FlowField& flow, int offset_x, int offset_y, int canvas_width,
                     int canvas_height) {  // flow.hpp:65-66
    if (offset_x < 0 || offset_y < 0 || offset_x + flow.width > canvas_width ||
        offset_y + flow.height > canvas_height)
        throw ContractError("embed_flow: crop box does not fit inside the canvas");
    FlowField out(canvas_width, canvas_height);
    check(fs_embed_flow(flow.vec.data(), flow.valid.data(), flow.width, flow.height, offset_x,
                        offset_y, canvas_width, canvas_height, out.vec.data(), out.valid.data(),
                        nullptr));
    return out;
}

// Middlebury .flo debug I/O (flow.hpp:68-71): host file plumbing, same format.
void write_flo(const FlowField& flow, const std::string& path) {
    std::ofstream f(path, std::ios::binary);
    if (!f) throw IoError("cannot open for writing: " + path);
    f.write("PIEH", 4);
    int32_t w = flow.width, h = flow.height;
    f.write(reinterpret_cast<const char*>(&w), 4);
    f.write(reinterpret_cast<const char*>(&h), 4);
    f.write(reinterpret_cast<const char*>(flow.vec.data()),
            static_cast<std::streamsize>(flow.vec.size() * sizeof(float)));
    if (!f) throw IoError("write failed: " + path);
}

FlowField read_flo(const std::string& path) {
    std::ifstream f(path, std::ios::binary);
    if (!f) throw IoError("cannot open for reading: " + path);
    char magic[4];
    f.read(magic, 4);
    if (!f || std::memcmp(magic, "PIEH", 4) != 0) throw FormatError("not a .flo file: " + path);
    int32_t w = 0, h = 0;
    f.read(reinterpret_cast<char*>(&w), 4);
    f.read(reinterpret_cast<char*>(&h), 4);
    if (!f || w < 1 || h < 1 || w > 99999 || h > 99999)
        throw FormatError("illegal .flo dimensions: " + path);
    FlowField flow(w, h);
    f.read(reinterpret_cast<char*>(flow.vec.data()),
           static_cast<std::streamsize>(flow.vec.size() * sizeof(float)));
    if (!f) throw FormatError("truncated .flo file: " + path);
    return flow;
}

// ---------------------------------------------------------------- blendfield
DistanceField distance_transform(const Mask& mask) {  // blend_field.hpp:32
    DistanceField out;
    out.width = mask.width;
    out.height = mask.height;
    out.d.resize(static_cast<size_t>(mask.width) * mask.height);
    check(fs_distance_transform(mask.v.data(), mask.width, mask.height, out.d.data(), nullptr));
    return out;
}

BlendField compute_blend(const RegionPartition& partition) {  // blend_field.hpp:34
    BlendField out;
    out.width = partition.width;
    out.height = partition.height;
    out.b.resize(static_cast<size_t>(partition.width) * partition.height);
    std::vector<uint8_t> label = labels_of(partition);
    int64_t counts[4];
    for (int r = 0; r < 4; ++r) counts[r] = partition.counts[r];
    if (!out.b.empty())
        check(fs_compute_blend(label.data(), counts, partition.width, partition.height,
                               out.b.data(), nullptr));
    return out;
}

// src/blend_field.cpp:132-137: lround(clamp(b, 0, 1) * 255.0) in double, gray
void save_blend_png(const BlendField& field, const std::string& path) {
    std::vector<uint8_t> bytes(static_cast<size_t>(field.width) * field.height);
    for (size_t k = 0; k < bytes.size(); ++k)
        bytes[k] = static_cast<uint8_t>(std::lround(std::clamp(field.b[k], 0.0, 1.0) * 255.0));
    detail::write_png(path, field.width, field.height, 1, bytes);
}

// ---------------------------------------------------------------- blender
void BlendParams::validate() const {  // src/blender.cpp:11-16
    if (!(k_softmax_sharpness > 0.0) || !std::isfinite(k_softmax_sharpness))
        throw ContractError("BlendParams: k_softmax_sharpness must be finite and > 0");
    if (k_flow_mag_coef < 0.0 || !std::isfinite(k_flow_mag_coef))
        throw ContractError("BlendParams: k_flow_mag_coef must be finite and >= 0");
}

std::pair<double, double> softmax_weights(double blend_l, double blend_r, double mag_rtol,
                                          double mag_ltor, const BlendParams& params) {
    fs_blend_params p = to_c(params);
    double sl = 0, sr = 0;
    fs_softmax_weights(blend_l, blend_r, mag_rtol, mag_ltor, &p, &sl, &sr);
    return {sl, sr};
}

namespace {
void check_canvas(const ImageBuf& L, const ImageBuf& R, const RegionPartition& partition) {
    if (L.width() != R.width() || L.height() != R.height() || L.width() != partition.width ||
        L.height() != partition.height || L.channels() != R.channels())
        throw ContractError("blend: canvas dimensions or channel counts differ");
}
}  // namespace

ImageBuf blend_pair(const ImageBuf& L, const ImageBuf& R, const FlowField& flowLtoR,
                    const FlowField& flowRtoL, const BlendField& blend,
                    const RegionPartition& partition, const BlendParams& params) {
    params.validate();
    check_canvas(L, R, partition);
    if (flowLtoR.width != partition.width || flowLtoR.height != partition.height ||
        flowRtoL.width != partition.width || flowRtoL.height != partition.height ||
        blend.width != partition.width || blend.height != partition.height)
        throw ContractError("blend_pair: flow or blend field dimensions differ from canvas");
    const int w = partition.width, h = partition.height;
    ImageBuf F(w, h, L.channels(), 0.0f, true);
    if (w == 0 || h == 0) return F;
    std::vector<uint8_t> vl = valid_bytes(L), vr = valid_bytes(R), label = labels_of(partition);
    std::vector<uint8_t> fv(static_cast<size_t>(w) * h);
    fs_blend_params p = to_c(params);
    check(fs_blend_pair(L.data().data(), vl.data(), R.data().data(), vr.data(), w, h, L.channels(),
                        flowLtoR.vec.data(), flowRtoL.vec.data(), blend.b.data(), label.data(), &p,
                        F.data().data(), fv.data(), nullptr));
    set_valid_bytes(F, fv);
    return F;
}

ImageBuf feather_blend(const ImageBuf& L, const ImageBuf& R, const BlendField& blend,
                       const RegionPartition& partition) {
    check_canvas(L, R, partition);
    if (blend.width != partition.width || blend.height != partition.height)
        throw ContractError("feather_blend: blend field dimensions differ from canvas");
    const int w = partition.width, h = partition.height;
    ImageBuf F(w, h, L.channels(), 0.0f, true);
    if (w == 0 || h == 0) return F;
    std::vector<uint8_t> vl = valid_bytes(L), vr = valid_bytes(R), label = labels_of(partition);
    std::vector<uint8_t> fv(static_cast<size_t>(w) * h);
    check(fs_feather_blend(L.data().data(), vl.data(), R.data().data(), vr.data(), w, h,
                           L.channels(), blend.b.data(), label.data(), F.data().data(), fv.data(),
                           nullptr));
    set_valid_bytes(F, fv);
    return F;
}

std::pair<ImageBuf, ImageBuf> warp_constituents(const ImageBuf& L, const ImageBuf& R,
                                                const FlowField& flowLtoR,
                                                const FlowField& flowRtoL,
                                                const BlendField& blend,
                                                const RegionPartition& partition) {
    check_canvas(L, R, partition);
    const int w = partition.width, h = partition.height;
    ImageBuf wl = L, wr = R;
    if (w == 0 || h == 0) return {wl, wr};
    std::vector<uint8_t> vl = valid_bytes(L), vr = valid_bytes(R), label = labels_of(partition);
    std::vector<uint8_t> ovl(vl.size()), ovr(vr.size());
    check(fs_warp_constituents(L.data().data(), vl.data(), R.data().data(), vr.data(), w, h,
                               L.channels(), flowLtoR.vec.data(), flowRtoL.vec.data(),
                               blend.b.data(), label.data(), wl.data().data(), ovl.data(),
                               wr.data().data(), ovr.data(), nullptr));
    set_valid_bytes(wl, ovl);
    set_valid_bytes(wr, ovr);
    return {std::move(wl), std::move(wr)};
}

// ---------------------------------------------------------------- runtime
// parallel.hpp:9-18.  The GPU path has no host worker pool; parallel_rows is
// still provided for host-side callers (e.g. the reference's metrics).
namespace {
std::atomic<int> g_threads{0};
}
void set_thread_count(int n) {
    g_threads.store(n < 0 ? 0 : n);
    fs_set_thread_count(n);
}
int thread_count() { return g_threads.load(); }
int resolved_thread_count() {
    int n = g_threads.load();
    if (n == 0)
        if (const char* s = std::getenv("FLOWSTITCH_THREADS")) n = std::max(0, std::atoi(s));
    if (n == 0) n = static_cast<int>(std::thread::hardware_concurrency());
    return std::max(1, n);
}
void parallel_rows(int rows, const std::function<void(int, int)>& fn) {
    int workers = std::min(resolved_thread_count(), rows);
    if (workers <= 1 || rows <= 1) {
        fn(0, rows);
        return;
    }
    std::vector<std::thread> pool;
    int chunk = (rows + workers - 1) / workers;
    for (int w = 1; w < workers; ++w) {
        int b = w * chunk, e = std::min(rows, b + chunk);
        if (b >= e) break;
        pool.emplace_back(fn, b, e);
    }
    fn(0, std::min(rows, chunk));
    for (auto& t : pool) t.join();
}

}  // namespace flowstitch
