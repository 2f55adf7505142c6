// flowstitch::b200::stitch_placed (include/flowstitch_b200.hpp).  (The PNG
// codec the reference's pipeline.cpp / image layer link against is
// png_codec.cpp.)
#include <chrono>
#include <cstring>
#include <vector>

#include "flowstitch/errors.hpp"
#include "flowstitch/pipeline.hpp"
#include "flowstitch_b200.hpp"
#include "fs_b200.h"
#include "png_io.hpp"

namespace flowstitch {
namespace b200 {

namespace {
void rethrow(fs_status st) {
    if (st == FS_OK) return;
    std::string msg = fs_last_error();
    if (st == FS_ERR_EMPTY_REGION) throw EmptyRegionError(msg);
    if (st == FS_ERR_LAYOUT) throw LayoutError(msg);
    if (st == FS_ERR_CONTRACT || st == FS_ERR_UNSUPPORTED) throw ContractError(msg);
    throw std::runtime_error("flowstitch-b200: " + msg);
}
std::vector<uint8_t> valid_of(const ImageBuf& img) {
    std::vector<uint8_t> v(static_cast<size_t>(img.width()) * img.height());
    for (int j = 0; j < img.height(); ++j)
        for (int i = 0; i < img.width(); ++i)
            v[static_cast<size_t>(j) * img.width() + i] = img.valid(i, j) ? 1 : 0;
    return v;
}
}  // namespace

// pipeline.hpp:75-77
TranslationEstimate estimate_translation(const ImageBuf& A, const ImageBuf& B, int max_shift) {
    if (A.channels() != 1 || B.channels() != 1)
        throw ContractError("estimate_translation: grayscale inputs required");
    if (A.width() != B.width() || A.height() != B.height())
        throw ContractError("estimate_translation: dimension mismatch");
    TranslationEstimate t;
    rethrow(fs_estimate_translation(A.data().data(), B.data().data(), A.width(), A.height(), 1,
                                    max_shift, &t.dx, &t.dy, &t.score, nullptr));
    return t;
}

// pipeline.hpp:81-83
double misalignment_score(const ImageBuf& L, const ImageBuf& R, const RegionPartition& partition,
                          int patch_radius, int stride) {
    if (L.width() != R.width() || L.height() != R.height() || L.width() != partition.width ||
        L.height() != partition.height)
        throw ContractError("misalignment_score: dimension mismatch");
    std::vector<uint8_t> label(partition.label.size());
    for (size_t k = 0; k < label.size(); ++k) label[k] = static_cast<uint8_t>(partition.label[k]);
    int64_t counts[4];
    for (int r = 0; r < 4; ++r) counts[r] = partition.counts[r];
    std::vector<uint8_t> vl = valid_of(L), vr = valid_of(R);
    double out = 0.0;
    if (L.channels() == R.channels()) {
        rethrow(fs_misalignment_score(L.data().data(), vl.data(), R.data().data(), vr.data(),
                                      L.width(), L.height(), L.channels(), label.data(), counts,
                                      patch_radius, stride, &out, nullptr));
        return out;
    }
    // mixed channel counts: both to gray first (the reference grays each)
    const size_t n = static_cast<size_t>(L.width()) * L.height();
    std::vector<float> gl(n), gr(n);
    rethrow(fs_to_gray(L.data().data(), L.width(), L.height(), L.channels(), gl.data(), nullptr));
    rethrow(fs_to_gray(R.data().data(), R.width(), R.height(), R.channels(), gr.data(), nullptr));
    rethrow(fs_misalignment_score(gl.data(), vl.data(), gr.data(), vr.data(), L.width(),
                                  L.height(), 1, label.data(), counts, patch_radius, stride, &out,
                                  nullptr));
    return out;
}

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
    rethrow(st);
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
