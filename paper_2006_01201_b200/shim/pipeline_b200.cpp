// flowstitch::b200::stitch_placed (include/flowstitch_b200.hpp) and the PNG
// codec entry points the reference's pipeline.cpp / image layer link against
// (proj/src/png_io.hpp) — PNG is host file plumbing outside the GPU path, so
// they report IoError.
#include <chrono>
#include <cstring>
#include <vector>

#include "flowstitch/errors.hpp"
#include "flowstitch/pipeline.hpp"
#include "flowstitch_b200.hpp"
#include "fs_b200.h"
#include "png_io.hpp"

namespace flowstitch {
namespace detail {
RawPng read_png(const std::string& path) {
    throw IoError("flowstitch-b200: PNG decoding is not part of the GPU path (" + path + ")");
}
void write_png(const std::string& path, int, int, int, const std::vector<uint8_t>&) {
    throw IoError("flowstitch-b200: PNG encoding is not part of the GPU path (" + path + ")");
}
void read_png_size(const std::string& path, int&, int&) {
    throw IoError("flowstitch-b200: PNG decoding is not part of the GPU path (" + path + ")");
}
}  // namespace detail

namespace b200 {

std::pair<ImageBuf, StitchReport> stitch_placed(const std::vector<PlacedImage>& placed,
                                                int canvas_width, int canvas_height,
                                                const FlowParams& flow_params,
                                                const BlendParams& blend_params) {
    if (placed.size() < 2) throw ContractError("stitch: at least two images required");
    flow_params.validate();
    blend_params.validate();
    const int n = static_cast<int>(placed.size());
    const int ch = placed[0].image.channels();
    for (const auto& p : placed)
        if (p.image.channels() != ch)
            throw ContractError("stitch: mixed grayscale and color inputs");
    auto t0 = std::chrono::steady_clock::now();
    std::vector<const float*> imgs(n);
    std::vector<std::vector<uint8_t>> valid(n);
    std::vector<const uint8_t*> vptr(n);
    std::vector<int> dims(2 * n), offs(2 * n);
    for (int k = 0; k < n; ++k) {
        const ImageBuf& im = placed[k].image;
        imgs[k] = im.data().data();
        valid[k].resize(static_cast<size_t>(im.width()) * im.height());
        for (int j = 0; j < im.height(); ++j)
            for (int i = 0; i < im.width(); ++i)
                valid[k][static_cast<size_t>(j) * im.width() + i] = im.valid(i, j) ? 1 : 0;
        vptr[k] = valid[k].data();
        dims[2 * k] = im.width();
        dims[2 * k + 1] = im.height();
        offs[2 * k] = placed[k].offset_x;
        offs[2 * k + 1] = placed[k].offset_y;
    }
    ImageBuf pano(canvas_width, canvas_height, ch, 0.0f, false);
    std::vector<uint8_t> pv(static_cast<size_t>(canvas_width) * canvas_height);
    std::vector<fs_pair_stats> stats(n - 1);
    fs_flow_params fp{flow_params.levels, flow_params.window_radius,
                      flow_params.iterations_per_level, flow_params.min_eigen_eps,
                      flow_params.smoothing_passes};
    fs_blend_params bp{blend_params.k_softmax_sharpness, blend_params.k_flow_mag_coef};
    fs_status st = fs_stitch_placed(n, imgs.data(), vptr.data(), dims.data(), offs.data(), ch,
                                    canvas_width, canvas_height, &fp, &bp, pano.data().data(),
                                    pv.data(), stats.data(), nullptr);
    if (st != FS_OK) {
        std::string msg = fs_last_error();
        if (st == FS_ERR_EMPTY_REGION) throw EmptyRegionError(msg);
        if (st == FS_ERR_LAYOUT) throw LayoutError(msg);
        if (st == FS_ERR_CONTRACT || st == FS_ERR_UNSUPPORTED) throw ContractError(msg);
        throw std::runtime_error("flowstitch-b200: " + msg);
    }
    for (int j = 0; j < canvas_height; ++j)
        for (int i = 0; i < canvas_width; ++i)
            pano.set_valid(i, j, pv[static_cast<size_t>(j) * canvas_width + i] != 0);
    StitchReport rep;
    for (const auto& s : stats) {
        PairStats ps;
        ps.overlap_pixels = static_cast<long>(s.overlap_pixels);
        ps.mean_flow_mag_ltor = s.mean_flow_mag_ltor;
        ps.mean_flow_mag_rtol = s.mean_flow_mag_rtol;
        ps.flow_seconds = s.flow_seconds;
        ps.blend_seconds = s.blend_seconds;
        if (s.misalignment_present & 1) ps.misalignment_before = s.misalignment_before;
        if (s.misalignment_present & 2) ps.misalignment_after = s.misalignment_after;
        rep.pairs.push_back(ps);
    }
    rep.total_seconds =
        std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return {std::move(pano), std::move(rep)};
}

}  // namespace b200
}  // namespace flowstitch
