// wavelift_b200_io.hpp -- the reference's file formats for the B200 drop-in
// (header-only, host C++17):
//
//  * binary PGM (P5), 8-bit and 16-bit big-endian samples, '#' comments in
//    the header; pixels map to [0, 1) as value / (maxval + 1) and back with
//    rounding and clamping (reference: proj/include/wavelift/pgm.hpp:1-30,
//    proj/src/pgm.cpp:42-103);
//  * the subband container "WAVELIFT-SUBBANDS 1": ASCII header lines
//    (wavelet, scheme, levels, boundary, scaling, image, one "level i w h"
//    line per level, "data") followed by raw little-endian float64 planes,
//    per level finest first HL, LH, HH, the coarsest level preceded by its LL
//    (reference: proj/include/wavelift/subband_io.hpp:7-20,
//    proj/src/subband_io.cpp:53-134).
//
// Same names and error behaviour as the reference (std::runtime_error on I/O
// failure or malformed content). Pyramid values are the float32 results of
// the GPU path widened to float64, so a file written here round-trips every
// plane bit-exactly, as the reference's does.
#ifndef WAVELIFT_B200_IO_HPP_
#define WAVELIFT_B200_IO_HPP_

#include <algorithm>
#include <cctype>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <fstream>
#include <sstream>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "wavelift_b200.hpp"

namespace wavelift {
inline namespace b200 {

static_assert(sizeof(double) == 8, "float64 payload");

struct PgmImage {
    int width = 0;
    int height = 0;
    int maxval = 255;  // < 256: 1-byte samples, else 2-byte big-endian
    std::vector<std::uint16_t> pixels;  // row-major
};

namespace io_detail {

// Next header token; skips whitespace and '#' comments to end of line.
inline std::string next_token(std::istream& in) {
    std::string tok;
    for (int ch = in.get(); ch != EOF; ch = in.get()) {
        if (ch == '#') {
            while ((ch = in.get()) != EOF && ch != '\n') {
            }
            continue;
        }
        if (std::isspace(ch)) {
            if (!tok.empty()) return tok;
            continue;
        }
        tok.push_back(static_cast<char>(ch));
    }
    return tok;
}

inline int positive(const std::string& tok, const char* what) {
    long v = 0;
    try {
        std::size_t used = 0;
        v = std::stol(tok, &used);
        if (used != tok.size()) v = 0;
    } catch (...) {
        v = 0;
    }
    if (v <= 0 || v > (1l << 20)) throw std::runtime_error(std::string("malformed PGM: bad ") + what);
    return static_cast<int>(v);
}

inline bool little_endian() {
    const std::uint16_t one = 1;
    unsigned char b;
    std::memcpy(&b, &one, 1);
    return b == 1;
}

inline void put_plane(std::ostream& out, const std::vector<double>& p, int w, int h) {
    if (p.size() != static_cast<std::size_t>(w) * h)
        throw std::runtime_error("subband plane has inconsistent dimensions");
    if (!little_endian()) throw std::runtime_error("raw float64 payload needs a little-endian host");
    out.write(reinterpret_cast<const char*>(p.data()),
              static_cast<std::streamsize>(p.size() * sizeof(double)));
}

inline std::vector<double> get_plane(std::istream& in, int w, int h) {
    std::vector<double> p(static_cast<std::size_t>(w) * h);
    in.read(reinterpret_cast<char*>(p.data()), static_cast<std::streamsize>(p.size() * 8));
    if (static_cast<std::size_t>(in.gcount()) != p.size() * 8)
        throw std::runtime_error("malformed subband file: truncated payload");
    return p;
}

inline std::string keyed(std::istream& in, const std::string& key) {
    std::string line;
    if (!std::getline(in, line) || line.compare(0, key.size() + 1, key + " ") != 0)
        throw std::runtime_error("malformed subband file: expected '" + key + "' line");
    return line.substr(key.size() + 1);
}

}  // namespace io_detail

inline PgmImage read_pgm(const std::string& path) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw std::runtime_error("cannot open " + path);
    if (io_detail::next_token(in) != "P5") throw std::runtime_error("malformed PGM: not binary P5");
    PgmImage img;
    img.width = io_detail::positive(io_detail::next_token(in), "width");
    img.height = io_detail::positive(io_detail::next_token(in), "height");
    img.maxval = io_detail::positive(io_detail::next_token(in), "maxval");
    if (img.maxval > 65535) throw std::runtime_error("malformed PGM: maxval > 65535");
    const std::size_t n = static_cast<std::size_t>(img.width) * img.height;
    const int bytes = img.maxval < 256 ? 1 : 2;
    std::vector<unsigned char> raw(n * bytes);
    in.read(reinterpret_cast<char*>(raw.data()), static_cast<std::streamsize>(raw.size()));
    if (static_cast<std::size_t>(in.gcount()) != raw.size())
        throw std::runtime_error("malformed PGM: truncated pixel data");
    img.pixels.resize(n);
    for (std::size_t i = 0; i < n; ++i) {
        const unsigned v = bytes == 1 ? raw[i] : (static_cast<unsigned>(raw[2 * i]) << 8) | raw[2 * i + 1];
        if (v > static_cast<unsigned>(img.maxval))
            throw std::runtime_error("malformed PGM: sample exceeds maxval");
        img.pixels[i] = static_cast<std::uint16_t>(v);
    }
    return img;
}

inline void write_pgm(const std::string& path, const PgmImage& img) {
    std::ofstream out(path, std::ios::binary);
    if (!out) throw std::runtime_error("cannot open " + path + " for writing");
    out << "P5\n" << img.width << " " << img.height << "\n" << img.maxval << "\n";
    const bool wide = img.maxval >= 256;
    for (std::uint16_t v : img.pixels) {
        if (wide) out.put(static_cast<char>(v >> 8));
        out.put(static_cast<char>(v & 0xff));
    }
    if (!out) throw std::runtime_error("failed writing " + path);
}

inline Image to_image(const PgmImage& pgm) {
    Image img(pgm.width, pgm.height);
    const double scale = 1.0 / (pgm.maxval + 1.0);
    for (std::size_t i = 0; i < pgm.pixels.size(); ++i) img.samples[i] = pgm.pixels[i] * scale;
    return img;
}

inline PgmImage from_image(const Image& img, int maxval = 255) {
    PgmImage pgm;
    pgm.width = img.width;
    pgm.height = img.height;
    pgm.maxval = maxval;
    pgm.pixels.resize(img.samples.size());
    for (std::size_t i = 0; i < img.samples.size(); ++i) {
        const double v = std::lround(img.samples[i] * (maxval + 1.0));
        pgm.pixels[i] = static_cast<std::uint16_t>(std::min<double>(std::max(v, 0.0), maxval));
    }
    return pgm;
}

struct SubbandHeader {
    std::string wavelet;
    std::string scheme;
    int levels = 1;
    BoundaryMode boundary = BoundaryMode::periodic;
    bool scaling = false;
    int image_w = 0;
    int image_h = 0;
};

inline void write_subbands(const std::string& path, const SubbandHeader& h, const Pyramid& p) {
    if (static_cast<int>(p.details.size()) != h.levels)
        throw std::runtime_error("pyramid level count does not match header");
    std::ofstream out(path, std::ios::binary);
    if (!out) throw std::runtime_error("cannot open " + path + " for writing");
    out << "WAVELIFT-SUBBANDS 1\n"
        << "wavelet " << h.wavelet << "\n"
        << "scheme " << h.scheme << "\n"
        << "levels " << h.levels << "\n"
        << "boundary " << boundary_name(h.boundary) << "\n"
        << "scaling " << (h.scaling ? 1 : 0) << "\n"
        << "image " << h.image_w << " " << h.image_h << "\n";
    for (int i = 0; i < h.levels; ++i)
        out << "level " << i + 1 << " " << p.details[i].w << " " << p.details[i].h << "\n";
    out << "data\n";
    for (int i = 0; i < h.levels; ++i) {
        const PyramidLevel& l = p.details[i];
        if (i == h.levels - 1) {
            if (p.ll_w != l.w || p.ll_h != l.h)
                throw std::runtime_error("coarsest LL plane has inconsistent dimensions");
            io_detail::put_plane(out, p.ll, l.w, l.h);
        }
        io_detail::put_plane(out, l.hl, l.w, l.h);
        io_detail::put_plane(out, l.lh, l.w, l.h);
        io_detail::put_plane(out, l.hh, l.w, l.h);
    }
    if (!out) throw std::runtime_error("failed writing " + path);
}

inline std::pair<SubbandHeader, Pyramid> read_subbands(const std::string& path) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw std::runtime_error("cannot open " + path);
    std::string line;
    if (!std::getline(in, line) || line != "WAVELIFT-SUBBANDS 1")
        throw std::runtime_error("malformed subband file: bad magic");
    SubbandHeader h;
    h.wavelet = io_detail::keyed(in, "wavelet");
    h.scheme = io_detail::keyed(in, "scheme");
    try {
        h.levels = std::stoi(io_detail::keyed(in, "levels"));
    } catch (const std::logic_error&) {
        h.levels = 0;
    }
    if (h.levels < 1) throw std::runtime_error("malformed subband file: bad levels");
    const auto b = parse_boundary(io_detail::keyed(in, "boundary"));
    if (!b) throw std::runtime_error("malformed subband file: bad boundary");
    h.boundary = *b;
    try {
        h.scaling = std::stoi(io_detail::keyed(in, "scaling")) != 0;
    } catch (const std::logic_error&) {
        throw std::runtime_error("malformed subband file: bad scaling");
    }
    {
        std::istringstream d(io_detail::keyed(in, "image"));
        if (!(d >> h.image_w >> h.image_h)) throw std::runtime_error("malformed subband file: bad image line");
    }
    Pyramid p;
    for (int i = 0; i < h.levels; ++i) {
        std::istringstream d(io_detail::keyed(in, "level"));
        int idx = 0;
        PyramidLevel l;
        if (!(d >> idx >> l.w >> l.h) || idx != i + 1 || l.w <= 0 || l.h <= 0)
            throw std::runtime_error("malformed subband file: bad level line");
        p.details.push_back(std::move(l));
    }
    if (!std::getline(in, line) || line != "data")
        throw std::runtime_error("malformed subband file: missing data marker");
    for (int i = 0; i < h.levels; ++i) {
        PyramidLevel& l = p.details[i];
        if (i == h.levels - 1) {
            p.ll_w = l.w;
            p.ll_h = l.h;
            p.ll = io_detail::get_plane(in, l.w, l.h);
        }
        l.hl = io_detail::get_plane(in, l.w, l.h);
        l.lh = io_detail::get_plane(in, l.w, l.h);
        l.hh = io_detail::get_plane(in, l.w, l.h);
    }
    return {std::move(h), std::move(p)};
}

}  // namespace b200
}  // namespace wavelift

#endif  // WAVELIFT_B200_IO_HPP_
