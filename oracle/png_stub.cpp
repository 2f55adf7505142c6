// TEST INFRASTRUCTURE (oracle) — not product code.
//
// Stand-in for the reference's libpng codec (proj/src/png_io.cpp:22-132), which
// cannot be built here: libpng headers are absent (proj/CMakeLists.txt:11).
// The flow/blend hot path never touches PNG; only load_image/save_image
// (proj/src/image.cpp:27-68), parse_layout (proj/src/pipeline.cpp:101) and
// save_blend_png (proj/src/blend_field.cpp:132-137) call into these, and the
// oracle never calls those. Every entry point throws IoError so an accidental
// call is loud.
#include <string>
#include <vector>

#include "flowstitch/errors.hpp"
#include "png_io.hpp"

namespace flowstitch::detail {

RawPng read_png(const std::string& path) {
    throw IoError("oracle png stub: PNG decoding is not built (" + path + ")");
}

void write_png(const std::string& path, int, int, int, const std::vector<uint8_t>&) {
    throw IoError("oracle png stub: PNG encoding is not built (" + path + ")");
}

void read_png_size(const std::string& path, int&, int&) {
    throw IoError("oracle png stub: PNG header reading is not built (" + path + ")");
}

} // namespace flowstitch::detail
