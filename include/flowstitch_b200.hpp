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
// panorama and exceptions; the report carries overlap pixels, mean flow
// magnitudes and device timings (the reference's misalignment metrics are
// evaluation helpers, not part of the fold, and are left empty).  A distinct
// name so it links next to the reference's pipeline.cpp.
std::pair<ImageBuf, StitchReport> stitch_placed(const std::vector<PlacedImage>& placed,
                                                int canvas_width, int canvas_height,
                                                const FlowParams& flow_params,
                                                const BlendParams& blend_params);

}  // namespace flowstitch::b200

#endif
