// flowstitch_b200.hpp — C++ entry points of the B200 drop-in beyond the
// reference's own headers.  Include after the reference's
// flowstitch/pipeline.hpp (the user's copy of the API this library replaces).
#ifndef FLOWSTITCH_B200_HPP
#define FLOWSTITCH_B200_HPP

#include <utility>
#include <vector>

#include "flowstitch/pipeline.hpp"

namespace flowstitch::b200 {

// Device-resident version of flowstitch::stitch_placed
// (proj/include/flowstitch/pipeline.hpp:64-67): the whole fold runs on the
// GPU through fs_stitch_placed (include/fs_b200.h).  Same inputs, same
// panorama, report (overlap pixels, mean flow magnitudes, misalignment
// before / after; timings are device times) and exceptions.  Distinct names
// so they link next to the reference's pipeline.cpp.
std::pair<ImageBuf, StitchReport> stitch_placed(const std::vector<PlacedImage>& placed,
                                                int canvas_width, int canvas_height,
                                                const FlowParams& flow_params,
                                                const BlendParams& blend_params);

// Device versions of the report helpers (pipeline.hpp:75-83), bit-identical.
TranslationEstimate estimate_translation(const ImageBuf& A, const ImageBuf& B, int max_shift);
double misalignment_score(const ImageBuf& L, const ImageBuf& R, const RegionPartition& partition,
                          int patch_radius = 8, int stride = 32);

}  // namespace flowstitch::b200

#endif
