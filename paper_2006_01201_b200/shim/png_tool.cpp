// PNG decode / encode through png_codec.cpp, for tests/test_png_io.py:
//   png_tool decode in.png out.raw      (out: "w h channels\n" + bytes)
//   png_tool encode w h channels in.raw out.png
//   png_tool size in.png                (prints "w h")
// Exit 2 on IoError / FormatError (message on stderr), 1 on usage errors.
#include <cstdio>
#include <fstream>
#include <iostream>
#include <iterator>
#include <string>
#include <vector>

#include "flowstitch/errors.hpp"
#include "png_io.hpp"

int main(int argc, char** argv) {
    using namespace flowstitch;
    try {
        const std::string cmd = argc > 1 ? argv[1] : "";
        if (cmd == "decode" && argc == 4) {
            detail::RawPng r = detail::read_png(argv[2]);
            std::ofstream o(argv[3], std::ios::binary);
            o << r.width << " " << r.height << " " << r.channels << "\n";
            o.write(reinterpret_cast<const char*>(r.bytes.data()), (std::streamsize)r.bytes.size());
            return 0;
        }
        if (cmd == "encode" && argc == 7) {
            std::ifstream i(argv[5], std::ios::binary);
            std::vector<uint8_t> b((std::istreambuf_iterator<char>(i)), std::istreambuf_iterator<char>());
            detail::write_png(argv[6], std::stoi(argv[2]), std::stoi(argv[3]), std::stoi(argv[4]), b);
            return 0;
        }
        if (cmd == "size" && argc == 3) {
            int w = 0, h = 0;
            detail::read_png_size(argv[2], w, h);
            std::cout << w << " " << h << "\n";
            return 0;
        }
    } catch (const IoError& e) {
        std::cerr << "error: " << e.what() << "\n";
        return 2;
    } catch (const FormatError& e) {
        std::cerr << "error: " << e.what() << "\n";
        return 2;
    }
    std::cerr << "usage: png_tool decode in.png out.raw | encode w h c in.raw out.png | size in.png\n";
    return 1;
}
