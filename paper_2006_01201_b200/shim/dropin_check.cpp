// Drop-in self-check (GPU): the B200 report helpers and fold against the
// reference's own pipeline.cpp, linked in the same binary.
//   flowstitch::misalignment_score / estimate_translation  (reference CPU code)
//   flowstitch::b200::misalignment_score / estimate_translation  (device)
//   flowstitch::stitch_placed  (reference orchestration over the drop-in
//   primitives) vs flowstitch::b200::stitch_placed  (device-resident fold)
#include <cmath>
#include <cstdio>
#include <vector>

#include "flowstitch/pipeline.hpp"
#include "flowstitch_b200.hpp"

using namespace flowstitch;

namespace {

// smooth multi-frequency texture in [0.1, 0.9], shifted by (sx, sy)
ImageBuf texture(int w, int h, int ch, double sx, double sy, int seed) {
    ImageBuf img(w, h, ch);
    for (int j = 0; j < h; ++j)
        for (int i = 0; i < w; ++i)
            for (int c = 0; c < ch; ++c) {
                double x = i - sx, y = j - sy, v = 0.0;
                for (int k = 1; k <= 6; ++k) {
                    double f = 0.05 * k + 0.013 * seed + 0.021 * c;
                    v += std::sin(f * x + 1.7 * k + seed) * std::cos(0.9 * f * y + 0.3 * k) / k;
                }
                img.set(i, j, c, static_cast<float>(0.5 + 0.18 * v));
            }
    return img;
}

int failures = 0;
void expect(bool ok, const char* what, double a, double b) {
    std::printf("%s %s: %.17g vs %.17g\n", ok ? "PASS" : "FAIL", what, a, b);
    if (!ok) ++failures;
}

}  // namespace

int main() {
    ImageBuf a = texture(160, 120, 1, 0, 0, 1), b = texture(160, 120, 1, 4, -3, 1);
    RegionPartition part = compute_partition(a.valid_mask(), b.valid_mask());
    double ref = misalignment_score(a, b, part, 8, 16), dev = b200::misalignment_score(a, b, part, 8, 16);
    expect(ref == dev, "misalignment_score gray", ref, dev);
    ImageBuf c = texture(200, 150, 3, 0, 0, 2), d = texture(200, 150, 3, -2, 5, 2);
    RegionPartition p2 = compute_partition(c.valid_mask(), d.valid_mask());
    ref = misalignment_score(c, d, p2);
    dev = b200::misalignment_score(c, d, p2);
    expect(ref == dev, "misalignment_score rgb", ref, dev);
    TranslationEstimate tr = estimate_translation(a, b, 8), td = b200::estimate_translation(a, b, 8);
    expect(tr.dx == td.dx && tr.dy == td.dy && tr.score == td.score, "estimate_translation",
           tr.score, td.score);

    ImageBuf v0 = texture(150, 100, 3, 0, 0, 3), v1 = texture(150, 100, 3, 110 - 3, 0, 3);
    std::vector<PlacedImage> placed = {{v0, 0, 0}, {v1, 110, 0}};
    FlowParams fp;
    fp.levels = 3;
    auto [pr, rr] = stitch_placed(placed, 260, 100, fp, BlendParams{});
    auto [pd, rd] = b200::stitch_placed(placed, 260, 100, fp, BlendParams{});
    double worst = 0.0;
    for (size_t k = 0; k < pr.data().size(); ++k)
        worst = std::max(worst, (double)std::fabs(pr.data()[k] - pd.data()[k]));
    expect(worst <= 1e-5, "stitch_placed max |d|", worst, 1e-5);
    const PairStats& s0 = rr.pairs[0];
    const PairStats& s1 = rd.pairs[0];
    expect(s0.overlap_pixels == s1.overlap_pixels, "overlap_pixels", s0.overlap_pixels,
           s1.overlap_pixels);
    expect(s0.misalignment_before.has_value() == s1.misalignment_before.has_value() &&
               (!s0.misalignment_before || *s0.misalignment_before == *s1.misalignment_before),
           "misalignment_before", s0.misalignment_before.value_or(-1),
           s1.misalignment_before.value_or(-1));
    expect(s0.misalignment_after.has_value() == s1.misalignment_after.has_value() &&
               (!s0.misalignment_after ||
                std::fabs(*s0.misalignment_after - *s1.misalignment_after) <= 1e-9),
           "misalignment_after", s0.misalignment_after.value_or(-1),
           s1.misalignment_after.value_or(-1));
    std::printf("%d check failure(s)\n", failures);
    return failures ? 1 : 0;
}
