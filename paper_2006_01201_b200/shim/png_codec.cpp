// 8-bit PNG codec for the drop-in's host file I/O: the entry points the
// reference's image layer and pipeline link against (proj/src/png_io.hpp:
// read_png, write_png, read_png_size), written on zlib (libpng is absent on
// this image).  Host plumbing, not part of the GPU path.
//
// Decoding produces what the reference's libpng set-up produces
// (proj/src/png_io.cpp:22-79): 8-bit samples; palette expanded to RGB;
// gray below 8 bits scaled to 8; a tRNS chunk turned into an alpha channel;
// gray+alpha promoted to RGBA; 1, 3 or 4 channels out; 16-bit and
// interlaced files refused with FormatError.  Encoding writes 8-bit gray /
// RGB / RGBA, non-interlaced, zlib level 6 (proj/src/png_io.cpp:81-115), each
// row filtered with the type of least absolute sum — fixed settings, so
// identical pixels give identical files.
#include <zlib.h>

#include <array>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "flowstitch/errors.hpp"
#include "png_io.hpp"

namespace flowstitch::detail {

namespace {

const uint8_t kSig[8] = {137, 'P', 'N', 'G', 13, 10, 26, 10};

struct FileCloser {
    void operator()(FILE* f) const {
        if (f) std::fclose(f);
    }
};
using File = std::unique_ptr<FILE, FileCloser>;

uint32_t be32(const uint8_t* p) {
    return (uint32_t(p[0]) << 24) | (uint32_t(p[1]) << 16) | (uint32_t(p[2]) << 8) | p[3];
}
void put32(std::vector<uint8_t>& o, uint32_t v) {
    o.push_back(uint8_t(v >> 24));
    o.push_back(uint8_t(v >> 16));
    o.push_back(uint8_t(v >> 8));
    o.push_back(uint8_t(v));
}

std::vector<uint8_t> slurp(const std::string& path) {
    File f(std::fopen(path.c_str(), "rb"));
    if (!f) throw IoError("cannot open for reading: " + path);
    std::vector<uint8_t> buf;
    uint8_t tmp[1 << 16];
    size_t n;
    while ((n = std::fread(tmp, 1, sizeof tmp, f.get())) > 0) buf.insert(buf.end(), tmp, tmp + n);
    return buf;
}

// PNG filter types 0..4 (PNG spec §9) on one row; bpp = bytes per pixel
uint8_t paeth(int a, int b, int c) {
    const int p = a + b - c, pa = std::abs(p - a), pb = std::abs(p - b), pc = std::abs(p - c);
    return uint8_t(pa <= pb && pa <= pc ? a : pb <= pc ? b : c);
}
void unfilter(uint8_t type, uint8_t* cur, const uint8_t* prev, size_t n, int bpp) {
    switch (type) {
        case 0: break;
        case 1:
            for (size_t i = bpp; i < n; ++i) cur[i] = uint8_t(cur[i] + cur[i - bpp]);
            break;
        case 2:
            for (size_t i = 0; i < n; ++i) cur[i] = uint8_t(cur[i] + prev[i]);
            break;
        case 3:
            for (size_t i = 0; i < n; ++i)
                cur[i] = uint8_t(cur[i] + ((i >= (size_t)bpp ? cur[i - bpp] : 0) + prev[i]) / 2);
            break;
        case 4:
            for (size_t i = 0; i < n; ++i)
                cur[i] = uint8_t(cur[i] + paeth(i >= (size_t)bpp ? cur[i - bpp] : 0, prev[i],
                                                i >= (size_t)bpp ? prev[i - bpp] : 0));
            break;
        default: throw FormatError("bad filter");
    }
}
uint8_t filtered(int type, const uint8_t* cur, const uint8_t* prev, size_t i, int bpp) {
    const int a = i >= (size_t)bpp ? cur[i - bpp] : 0, b = prev[i],
              c = i >= (size_t)bpp ? prev[i - bpp] : 0;
    switch (type) {
        case 1: return uint8_t(cur[i] - a);
        case 2: return uint8_t(cur[i] - b);
        case 3: return uint8_t(cur[i] - (a + b) / 2);
        case 4: return uint8_t(cur[i] - paeth(a, b, c));
        default: return cur[i];
    }
}

}  // namespace

RawPng read_png(const std::string& path) {
    const std::vector<uint8_t> f = slurp(path);
    if (f.size() < 8 || std::memcmp(f.data(), kSig, 8) != 0)
        throw FormatError("not a PNG file: " + path);
    auto bad = [&]() -> FormatError { return FormatError("PNG decode error: " + path); };
    uint32_t w = 0, h = 0;
    int depth = 0, ctype = -1, interlace = 0;
    std::vector<uint8_t> plte, trns, idat;
    bool have_ihdr = false, end = false;
    size_t pos = 8;
    while (!end) {
        if (pos + 12 > f.size()) throw bad();
        const uint32_t len = be32(&f[pos]);
        if (len > f.size() - pos - 12) throw bad();
        const uint8_t* type = &f[pos + 4];
        const uint8_t* data = &f[pos + 8];
        if (crc32(crc32(0L, Z_NULL, 0), type, len + 4) != be32(data + len)) throw bad();
        if (!std::memcmp(type, "IHDR", 4)) {
            if (len != 13) throw bad();
            w = be32(data);
            h = be32(data + 4);
            depth = data[8];
            ctype = data[9];
            interlace = data[12];
            if (data[10] != 0 || data[11] != 0) throw bad();
            have_ihdr = true;
        } else if (!std::memcmp(type, "PLTE", 4)) {
            plte.assign(data, data + len);
        } else if (!std::memcmp(type, "tRNS", 4)) {
            trns.assign(data, data + len);
        } else if (!std::memcmp(type, "IDAT", 4)) {
            idat.insert(idat.end(), data, data + len);
        } else if (!std::memcmp(type, "IEND", 4)) {
            end = true;
        } else if (!(type[0] & 0x20)) {  // unknown critical chunk
            throw bad();
        }
        pos += 12 + len;
    }
    if (!have_ihdr || w == 0 || h == 0 || w > (1u << 24) || h > (1u << 24)) throw bad();
    if (depth == 16) throw FormatError("16-bit PNG not supported: " + path);
    if (interlace != 0) throw FormatError("interlaced PNG not supported: " + path);
    int spp;  // samples per pixel of the stored format
    switch (ctype) {
        case 0: spp = 1; break;
        case 2: spp = 3; break;
        case 3: spp = 1; break;
        case 4: spp = 2; break;
        case 6: spp = 4; break;
        default: throw bad();
    }
    const bool depth_ok = depth == 8 || ((ctype == 0 || ctype == 3) &&
                                         (depth == 1 || depth == 2 || depth == 4));
    if (!depth_ok || (ctype == 3 && plte.empty())) throw bad();
    const size_t bits = (size_t)spp * depth;
    const size_t stride = ((size_t)w * bits + 7) / 8;
    const int bpp = (int)std::max<size_t>(1, bits / 8);
    std::vector<uint8_t> raw((stride + 1) * h);
    uLongf rl = raw.size();
    if (uncompress(raw.data(), &rl, idat.data(), idat.size()) != Z_OK || rl != raw.size())
        throw bad();
    std::vector<uint8_t> zero(stride, 0);
    for (uint32_t y = 0; y < h; ++y) {
        uint8_t* row = &raw[y * (stride + 1)];
        const uint8_t* prev = y ? &raw[(y - 1) * (stride + 1) + 1] : zero.data();
        try {
            unfilter(row[0], row + 1, prev, stride, bpp);
        } catch (const FormatError&) {
            throw bad();
        }
    }
    // output channels (the reference's transforms, proj/src/png_io.cpp:45-65)
    int out_ch;
    if (ctype == 3)
        out_ch = trns.empty() ? 3 : 4;
    else if (ctype == 0)
        out_ch = trns.size() >= 2 ? 4 : 1;  // gray + tRNS -> gray+alpha -> RGBA
    else if (ctype == 2)
        out_ch = trns.size() >= 6 ? 4 : 3;
    else
        out_ch = 4;  // gray+alpha promoted to RGBA; RGBA
    RawPng out;
    out.width = (int)w;
    out.height = (int)h;
    out.channels = out_ch;
    out.bytes.resize((size_t)w * h * out_ch);
    const int maxv = (1 << depth) - 1;
    for (uint32_t y = 0; y < h; ++y) {
        const uint8_t* row = &raw[y * (stride + 1) + 1];
        uint8_t* o = &out.bytes[(size_t)y * w * out_ch];
        for (uint32_t x = 0; x < w; ++x, o += out_ch) {
            if (ctype == 0 || ctype == 3) {
                unsigned v;
                if (depth == 8) {
                    v = row[x];
                } else {
                    const size_t bit = (size_t)x * depth;
                    v = (row[bit / 8] >> (8 - depth - bit % 8)) & maxv;
                }
                if (ctype == 3) {
                    if (3 * v + 2 >= plte.size()) throw bad();
                    o[0] = plte[3 * v];
                    o[1] = plte[3 * v + 1];
                    o[2] = plte[3 * v + 2];
                    if (out_ch == 4) o[3] = v < trns.size() ? trns[v] : 255;
                } else {
                    const uint8_t g = uint8_t(v * 255 / maxv);
                    if (out_ch == 1) {
                        o[0] = g;
                    } else {
                        const unsigned key = ((unsigned)trns[0] << 8 | trns[1]) & maxv;
                        o[0] = o[1] = o[2] = g;
                        o[3] = v == key ? 0 : 255;
                    }
                }
            } else if (ctype == 2) {
                const uint8_t* p = row + 3 * x;
                o[0] = p[0];
                o[1] = p[1];
                o[2] = p[2];
                if (out_ch == 4)
                    o[3] = (p[0] == trns[1] && p[1] == trns[3] && p[2] == trns[5]) ? 0 : 255;
            } else if (ctype == 4) {
                o[0] = o[1] = o[2] = row[2 * x];
                o[3] = row[2 * x + 1];
            } else {
                std::memcpy(o, row + 4 * x, 4);
            }
        }
    }
    return out;
}

void write_png(const std::string& path, int width, int height, int channels,
               const std::vector<uint8_t>& bytes) {
    if (width <= 0 || height <= 0 || (channels != 1 && channels != 3 && channels != 4) ||
        bytes.size() != (size_t)width * height * channels)
        throw IoError("PNG encode error: " + path);
    const size_t stride = (size_t)width * channels;
    std::vector<uint8_t> filt((stride + 1) * height);
    std::vector<uint8_t> zero(stride, 0), cand(stride);
    for (int y = 0; y < height; ++y) {
        const uint8_t* cur = &bytes[(size_t)y * stride];
        const uint8_t* prev = y ? cur - stride : zero.data();
        int best = 0;
        unsigned long best_sum = ~0ul;
        for (int t = 0; t < 5; ++t) {  // least sum of |signed residual|
            unsigned long sum = 0;
            for (size_t i = 0; i < stride; ++i) {
                const int8_t v = (int8_t)filtered(t, cur, prev, i, channels);
                sum += (unsigned long)std::abs((int)v);
            }
            if (sum < best_sum) {
                best_sum = sum;
                best = t;
            }
        }
        uint8_t* o = &filt[(size_t)y * (stride + 1)];
        o[0] = uint8_t(best);
        for (size_t i = 0; i < stride; ++i) o[1 + i] = filtered(best, cur, prev, i, channels);
    }
    uLongf zl = compressBound(filt.size());
    std::vector<uint8_t> z(zl);
    if (compress2(z.data(), &zl, filt.data(), filt.size(), 6) != Z_OK)
        throw IoError("PNG encode error: " + path);
    z.resize(zl);
    std::vector<uint8_t> png(kSig, kSig + 8);
    auto chunk = [&](const char* type, const uint8_t* data, size_t len) {
        put32(png, (uint32_t)len);
        const size_t at = png.size();
        png.insert(png.end(), type, type + 4);
        png.insert(png.end(), data, data + len);
        put32(png, (uint32_t)crc32(crc32(0L, Z_NULL, 0), &png[at], (uInt)(len + 4)));
    };
    std::vector<uint8_t> ihdr;
    put32(ihdr, (uint32_t)width);
    put32(ihdr, (uint32_t)height);
    ihdr.push_back(8);
    ihdr.push_back(uint8_t(channels == 1 ? 0 : channels == 3 ? 2 : 6));
    ihdr.push_back(0);
    ihdr.push_back(0);
    ihdr.push_back(0);
    chunk("IHDR", ihdr.data(), ihdr.size());
    chunk("IDAT", z.data(), z.size());
    chunk("IEND", nullptr, 0);
    File f(std::fopen(path.c_str(), "wb"));
    if (!f) throw IoError("cannot open for writing: " + path);
    if (std::fwrite(png.data(), 1, png.size(), f.get()) != png.size())
        throw IoError("PNG encode error: " + path);
}

void read_png_size(const std::string& path, int& width, int& height) {
    File f(std::fopen(path.c_str(), "rb"));
    if (!f) throw IoError("cannot open for reading: " + path);
    uint8_t head[24];
    if (std::fread(head, 1, 24, f.get()) != 24 || std::memcmp(head, kSig, 8) != 0)
        throw FormatError("not a PNG file: " + path);
    if (std::memcmp(head + 12, "IHDR", 4) != 0) throw FormatError("malformed PNG header: " + path);
    width = (int)be32(head + 16);
    height = (int)be32(head + 20);
}

}  // namespace flowstitch::detail
