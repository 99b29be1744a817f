// TEST INFRASTRUCTURE -- C-ABI shim over the UNMODIFIED reference library.
//
// Compiled together with /root/reference/proj/src/{laurent,polyphase,
// wavelets,schemes,transform}.cpp (see oracle/Makefile) into
// oracle/_ref/libwavelift_ref.so. Only tests/, __graft_entry__.smoke() and
// bench.py's CPU-baseline / reference arm load it, always as the checker or
// as the timed reference, never as the product. No reference source is
// copied: this file only calls the reference's public API
// (transform.hpp:47-95, schemes.hpp:29-84, wavelets.hpp:32, polyphase.hpp:58).
//
// Enum encodings shared with include/wl_dwt.h:
//   wavelet  0 cdf53, 1 cdf97, 2 dd137          (wavelets.cpp:27-62)
//   scheme   SchemeKind declaration order 0..9  (schemes.hpp:15-26)
//   boundary 0 periodic, 1 symmetric            (transform.hpp:44)
// Status: 0 ok, 1 std::invalid_argument, 2 any other exception.

#include "wavelift/pgm.hpp"
#include "wavelift/polyphase.hpp"
#include "wavelift/schemes.hpp"
#include "wavelift/subband_io.hpp"
#include "wavelift/transform.hpp"
#include "wavelift/wavelets.hpp"

#include <cstdio>
#include <cstring>
#include <random>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

using namespace wavelift;

namespace {

thread_local std::string g_err;

const char* wavelet_name(int w) {
    switch (w) {
        case 0: return "cdf53";
        case 1: return "cdf97";
        case 2: return "dd137";
    }
    throw std::invalid_argument("unknown wavelet id");
}

SchemeKind scheme_kind(int s) {
    if (s < 0 || s > 9) throw std::invalid_argument("unknown scheme id");
    return all_scheme_kinds()[static_cast<std::size_t>(s)];
}

BoundaryMode boundary_mode(int b) {
    if (b == 0) return BoundaryMode::periodic;
    if (b == 1) return BoundaryMode::symmetric;
    throw std::invalid_argument("unknown boundary id");
}

template <typename Fn>
int guarded(Fn&& fn) {
    try {
        fn();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 2;
    }
}

Image to_image(const double* px, int w, int h) {
    Image img;
    img.width = w;
    img.height = h;
    img.samples.assign(px, px + static_cast<std::size_t>(w > 0 ? w : 0) * (h > 0 ? h : 0));
    return img;
}

void put_quad(const QuadGrid& q, double* out4) {
    const std::size_t n = static_cast<std::size_t>(q.w) * q.h;
    for (int c = 0; c < 4; ++c) std::memcpy(out4 + c * n, q.planes[c].data(), n * sizeof(double));
}

QuadGrid get_quad(const double* in4, int qw, int qh) {
    QuadGrid q(qw, qh);
    const std::size_t n = static_cast<std::size_t>(qw) * qh;
    for (int c = 0; c < 4; ++c) q.planes[c].assign(in4 + c * n, in4 + (c + 1) * n);
    return q;
}

void json_poly2(std::ostringstream& os, const LaurentPoly2& p) {
    os << "[";
    bool first = true;
    for (const auto& [e, c] : p.terms()) {  // std::map order == summation order
        if (!first) os << ",";
        first = false;
        char buf[64];
        std::snprintf(buf, sizeof buf, "%.17g", c.to_double());
        os << "[" << e.first << "," << e.second << ",\"" << c.str() << "\"," << buf << "]";
    }
    os << "]";
}

}  // namespace

extern "C" {

const char* wlref_last_error() { return g_err.c_str(); }

int wlref_worker_count() { return worker_count(); }

// transform.cpp:163-176 forward(); out4 = LL,HL,LH,HH planes of (w/2)x(h/2).
int wlref_forward(const double* img, int w, int h, int wavelet, int scheme, int boundary,
                  int scaling, double* out4) {
    return guarded([&] {
        const Scheme s = build_scheme(scheme_kind(scheme), get_wavelet(wavelet_name(wavelet)));
        const QuadGrid q = forward(to_image(img, w, h), s, boundary_mode(boundary), scaling != 0);
        put_quad(q, out4);
    });
}

// transform.cpp:178-196 inverse(): wavelet-only (reversed negated Sweldens).
int wlref_inverse(const double* in4, int qw, int qh, int wavelet, int boundary, int undo_scaling,
                  double* img_out) {
    return guarded([&] {
        const Image img = inverse(get_quad(in4, qw, qh), get_wavelet(wavelet_name(wavelet)),
                                  boundary_mode(boundary), undo_scaling != 0);
        std::memcpy(img_out, img.samples.data(), img.samples.size() * sizeof(double));
    });
}

// transform.cpp:198-227. Flat layout: per level (finest first) HL,LH,HH of
// that level's plane size, then the coarsest LL.
int wlref_pyramid_forward(const double* img, int w, int h, int wavelet, int scheme, int levels,
                          int boundary, int scaling, double* out) {
    return guarded([&] {
        const Scheme s = build_scheme(scheme_kind(scheme), get_wavelet(wavelet_name(wavelet)));
        const Pyramid p =
            multi_level_forward(to_image(img, w, h), s, levels, boundary_mode(boundary), scaling != 0);
        double* o = out;
        for (const PyramidLevel& l : p.details) {
            for (const auto* v : {&l.hl, &l.lh, &l.hh}) {
                std::memcpy(o, v->data(), v->size() * sizeof(double));
                o += v->size();
            }
        }
        std::memcpy(o, p.ll.data(), p.ll.size() * sizeof(double));
    });
}

// transform.cpp:229-256 multi_level_inverse() on the flat layout above.
int wlref_pyramid_inverse(const double* in, int w, int h, int levels, int wavelet, int boundary,
                          int undo_scaling, double* img_out) {
    return guarded([&] {
        Pyramid p;
        const double* src = in;
        int pw = w / 2, ph = h / 2;
        for (int l = 0; l < levels; ++l) {
            PyramidLevel lev;
            lev.w = pw;
            lev.h = ph;
            const std::size_t n = static_cast<std::size_t>(pw) * ph;
            lev.hl.assign(src, src + n);
            lev.lh.assign(src + n, src + 2 * n);
            lev.hh.assign(src + 2 * n, src + 3 * n);
            src += 3 * n;
            p.details.push_back(std::move(lev));
            if (l + 1 < levels) {
                pw /= 2;
                ph /= 2;
            }
        }
        p.ll_w = pw;
        p.ll_h = ph;
        p.ll.assign(src, src + static_cast<std::size_t>(pw) * ph);
        const Image img =
            multi_level_inverse(p, get_wavelet(wavelet_name(wavelet)), boundary_mode(boundary),
                                undo_scaling != 0);
        std::memcpy(img_out, img.samples.data(), img.samples.size() * sizeof(double));
    });
}

// Applies one arbitrary real-mode step matrix with the reference's
// apply_step (transform.cpp:100-125). Taps: n rows of
// (dst, src, km, kn, coeff); entries not listed are zero except that a
// diagonal entry with no listed tap is the identity.
int wlref_apply_step(const double* in4, int qw, int qh, const int* tap_idx, const double* coeff,
                     int ntaps, int boundary, double* out4) {
    return guarded([&] {
        StepMatrix m(CoeffMode::real);
        LaurentPoly2 entries[16];
        bool touched[16] = {};
        for (int i = 0; i < 16; ++i) entries[i] = LaurentPoly2::zero(CoeffMode::real);
        for (int t = 0; t < ntaps; ++t) {
            const int d = tap_idx[4 * t], s = tap_idx[4 * t + 1];
            const int km = tap_idx[4 * t + 2], kn = tap_idx[4 * t + 3];
            LaurentPoly2& e = entries[d * 4 + s];
            e.set_term(km, kn, e.at(km, kn) + Coeff::real(coeff[t]));
            touched[d * 4 + s] = true;
        }
        for (int i = 0; i < 16; ++i)
            if (touched[i] || i / 4 != i % 4) m.set_entry(i / 4, i % 4, entries[i]);
        const QuadGrid out = apply_step(get_quad(in4, qw, qh), m, boundary_mode(boundary));
        put_quad(out, out4);
    });
}

int wlref_cost(int wavelet, int scheme, int* barriers, long* macs) {
    return guarded([&] {
        const Scheme s = build_scheme(scheme_kind(scheme), get_wavelet(wavelet_name(wavelet)));
        *barriers = count_barriers(s);
        *macs = count_macs(s);
    });
}

// JSON dump of build_scheme() (schemes.cpp:146-174): step labels, barrier
// flags and every 4x4 entry as [km, kn, "exact-or-real str", double] terms,
// plus the wavelet's zeta and, for Convolution, the four 2-D filters.
// Returns the needed buffer size (excluding NUL); writes when buflen allows.
long wlref_dump_scheme(int wavelet, int scheme, char* buf, long buflen) {
    std::string text;
    const int st = guarded([&] {
        const WaveletSpec w = get_wavelet(wavelet_name(wavelet));
        const Scheme s = build_scheme(scheme_kind(scheme), w);
        std::ostringstream os;
        char zbuf[64];
        std::snprintf(zbuf, sizeof zbuf, "%.17g", w.zeta);
        os << "{\"wavelet\":\"" << w.name << "\",\"scheme\":\"" << scheme_name(s.kind)
           << "\",\"zeta\":" << zbuf << ",\"exact\":" << (w.mode() == CoeffMode::exact ? 1 : 0)
           << ",\"barriers\":" << count_barriers(s) << ",\"macs\":" << count_macs(s)
           << ",\"steps\":[";
        for (std::size_t i = 0; i < s.steps.size(); ++i) {
            const Step& step = s.steps[i];
            if (i) os << ",";
            os << "{\"label\":\"" << step.label << "\",\"barrier\":" << (step.needs_barrier ? 1 : 0)
               << ",\"kind\":\"" << to_string(step.matrix.kind()) << "\",\"entries\":[";
            bool first = true;
            for (int r = 0; r < 4; ++r)
                for (int c = 0; c < 4; ++c) {
                    const LaurentPoly2& e = step.matrix.entry(r, c);
                    if (e.is_zero()) continue;
                    if (!first) os << ",";
                    first = false;
                    os << "[" << r << "," << c << ",";
                    json_poly2(os, e);
                    os << "]";
                }
            os << "]}";
        }
        os << "]";
        if (s.conv_filters) {
            os << ",\"conv\":[";
            const LaurentPoly2* f[4] = {&s.conv_filters->f_ll, &s.conv_filters->f_hl,
                                        &s.conv_filters->f_lh, &s.conv_filters->f_hh};
            for (int k = 0; k < 4; ++k) {
                if (k) os << ",";
                json_poly2(os, *f[k]);
            }
            os << "]";
        }
        os << "}";
        text = os.str();
    });
    if (st != 0) return -1;
    if (buf && buflen > static_cast<long>(text.size())) {
        std::memcpy(buf, text.c_str(), text.size() + 1);
    }
    return static_cast<long>(text.size());
}

// Restates the two image generators of proj/tests/test_util.hpp:58-74 with
// the same std:: engine and distributions, so fixtures equal the reference
// tests' own inputs (the distribution output is libstdc++-specific).
void wlref_random_image(int w, int h, unsigned seed, int dyadic, double* out) {
    std::mt19937 rng(seed);
    const std::size_t n = static_cast<std::size_t>(w) * h;
    if (dyadic) {
        std::uniform_int_distribution<int> dist(0, 255);
        for (std::size_t i = 0; i < n; ++i) out[i] = dist(rng) / 256.0;
    } else {
        std::uniform_real_distribution<double> dist(0.0, 1.0);
        for (std::size_t i = 0; i < n; ++i) out[i] = dist(rng);
    }
}

// Verification identity (polyphase.cpp:192-219 / schemes.cpp:230-236):
// max deviation of the scheme's step product from the reference matrix.
int wlref_verify_identity(int wavelet, int scheme, double* max_dev, int* match) {
    return guarded([&] {
        const WaveletSpec w = get_wavelet(wavelet_name(wavelet));
        const Scheme s = build_scheme(scheme_kind(scheme), w);
        const IdentityReport rep = verify_scheme_identity(
            scheme_step_matrices(s), scheme_reference_matrix(w),
            w.mode() == CoeffMode::exact ? 0.0 : 1e-12);
        *max_dev = rep.max_deviation;
        *match = rep.match ? 1 : 0;
    });
}


// ---- file formats (pgm.cpp, subband_io.cpp) and the CLI's cmd_transform
// (wavelift_main.cpp:153-177), through the unmodified reference library.
// Pyramids cross the ABI in the B200 flat layout: per level HL, LH, HH
// (finest first), then the coarsest LL.

int wlref_write_pgm(const char* path, int w, int h, int maxval, const unsigned short* px) {
    return guarded([&] {
        PgmImage p;
        p.width = w;
        p.height = h;
        p.maxval = maxval;
        p.pixels.assign(px, px + static_cast<std::size_t>(w) * h);
        write_pgm(path, p);
    });
}

// Two-call pattern: px may be null to query the size.
int wlref_read_pgm(const char* path, int* w, int* h, int* maxval, unsigned short* px) {
    return guarded([&] {
        const PgmImage p = read_pgm(path);
        *w = p.width;
        *h = p.height;
        *maxval = p.maxval;
        if (px) std::memcpy(px, p.pixels.data(), p.pixels.size() * sizeof(unsigned short));
    });
}

static Pyramid pyramid_from_flat(const double* flat, int w, int h, int levels) {
    Pyramid p;
    std::size_t off = 0;
    for (int l = 0; l < levels; ++l) {
        PyramidLevel lv;
        lv.w = w >> (l + 1);
        lv.h = h >> (l + 1);
        const std::size_t n = static_cast<std::size_t>(lv.w) * lv.h;
        lv.hl.assign(flat + off, flat + off + n);
        lv.lh.assign(flat + off + n, flat + off + 2 * n);
        lv.hh.assign(flat + off + 2 * n, flat + off + 3 * n);
        off += 3 * n;
        p.details.push_back(std::move(lv));
    }
    p.ll_w = w >> levels;
    p.ll_h = h >> levels;
    p.ll.assign(flat + off, flat + off + static_cast<std::size_t>(p.ll_w) * p.ll_h);
    return p;
}

int wlref_write_subbands(const char* path, const char* wavelet, const char* scheme, int levels,
                         int boundary, int scaling, int w, int h, const double* flat) {
    return guarded([&] {
        SubbandHeader hd;
        hd.wavelet = wavelet;
        hd.scheme = scheme;
        hd.levels = levels;
        hd.boundary = boundary_mode(boundary);
        hd.scaling = scaling != 0;
        hd.image_w = w;
        hd.image_h = h;
        write_subbands(path, hd, pyramid_from_flat(flat, w, h, levels));
    });
}

// header out-params; flat (w*h doubles) may be null to query the header.
int wlref_read_subbands(const char* path, char* wavelet64, char* scheme64, int* levels,
                        int* boundary, int* scaling, int* w, int* h, double* flat) {
    return guarded([&] {
        const auto [hd, p] = read_subbands(path);
        std::snprintf(wavelet64, 64, "%s", hd.wavelet.c_str());
        std::snprintf(scheme64, 64, "%s", hd.scheme.c_str());
        *levels = hd.levels;
        *boundary = hd.boundary == BoundaryMode::periodic ? 0 : 1;
        *scaling = hd.scaling ? 1 : 0;
        *w = hd.image_w;
        *h = hd.image_h;
        if (!flat) return;
        std::size_t off = 0;
        for (const PyramidLevel& lv : p.details)
            for (const auto* pl : {&lv.hl, &lv.lh, &lv.hh}) {
                std::memcpy(flat + off, pl->data(), pl->size() * sizeof(double));
                off += pl->size();
            }
        std::memcpy(flat + off, p.ll.data(), p.ll.size() * sizeof(double));
    });
}

// cmd_transform without --pad: PGM -> multi_level_forward -> subband file.
int wlref_transform_file(const char* in, const char* out, int wavelet, int scheme, int levels,
                         int boundary, int scaling) {
    return guarded([&] {
        const Image img = wavelift::to_image(read_pgm(in));
        const WaveletSpec wv = get_wavelet(wavelet_name(wavelet));
        const SchemeKind kind = scheme_kind(scheme);
        const Pyramid p = multi_level_forward(img, build_scheme(kind, wv), levels,
                                              boundary_mode(boundary), scaling != 0);
        SubbandHeader hd;
        hd.wavelet = wv.name;
        hd.scheme = scheme_name(kind);
        hd.levels = levels;
        hd.boundary = boundary_mode(boundary);
        hd.scaling = scaling != 0;
        hd.image_w = img.width;
        hd.image_h = img.height;
        write_subbands(out, hd, p);
    });
}

}  // extern "C"
