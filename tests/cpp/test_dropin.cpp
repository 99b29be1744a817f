// C++ parity test of the drop-in API (include/wavelift_b200.hpp) against the
// UNMODIFIED reference library (oracle/_ref/libwavelift_ref.so, C-ABI of
// oracle/ref_capi.cpp), modelled on proj/tests/test_transform.cpp.
// Built and run by tests/test_cpp_dropin.py on a GPU box. Exit 0 = all pass.
#include <cmath>
#include <cstdio>
#include <random>
#include <stdexcept>
#include <vector>

#include "wavelift_b200.hpp"

extern "C" {
int wlref_forward(const double*, int, int, int, int, int, int, double*);
int wlref_inverse(const double*, int, int, int, int, int, double*);
void wlref_random_image(int, int, unsigned, int, double*);
}

using namespace wavelift;

static int g_fail = 0, g_checks = 0;
#define CHECK(cond, ...)                                      \
    do {                                                      \
        ++g_checks;                                           \
        if (!(cond)) {                                        \
            ++g_fail;                                         \
            std::printf("FAIL %s:%d ", __FILE__, __LINE__);   \
            std::printf(__VA_ARGS__);                         \
            std::printf("\n");                                \
        }                                                     \
    } while (0)

static Image ref_image(int w, int h, unsigned seed, bool dyadic) {
    Image img(w, h);
    wlref_random_image(w, h, seed, dyadic ? 1 : 0, img.samples.data());
    return img;
}

static double rel_diff(const QuadGrid& a, const std::vector<double>& ref) {
    const std::size_t n = static_cast<std::size_t>(a.w) * a.h;
    double worst = 0;
    for (int c = 0; c < 4; ++c) {
        double lo = 1e300, hi = -1e300, m = 0;
        for (std::size_t i = 0; i < n; ++i) {
            lo = std::min(lo, ref[c * n + i]);
            hi = std::max(hi, ref[c * n + i]);
            m = std::max(m, std::abs(a.planes[c][i] - ref[c * n + i]));
        }
        const double range = hi - lo > 1e-12 ? hi - lo : 1.0;
        worst = std::max(worst, m / range);
    }
    return worst;
}

int main() {
    // test_transform.cpp:127-154 cross-scheme / reference parity (dyadic 32x32
    // seed 101 bit-exact for cdf53; uniform seed 102 within 1e-5 for cdf97).
    for (const char* wn : {"cdf53", "cdf97"}) {
        const WaveletSpec w = get_wavelet(wn);
        const bool exact = w.id == WL_CDF53;
        for (auto [iw, ih] : {std::pair{32, 32}, std::pair{256, 192}, std::pair{6, 4}}) {
            const Image img = ref_image(iw, ih, exact ? 101 : 102, exact);
            for (SchemeKind k : all_scheme_kinds())
                for (BoundaryMode b : {BoundaryMode::periodic, BoundaryMode::symmetric}) {
                    const QuadGrid got = forward(img, build_scheme(k, w), b, false);
                    std::vector<double> ref(img.samples.size());
                    wlref_forward(img.samples.data(), iw, ih, w.id, static_cast<int>(k),
                                  b == BoundaryMode::periodic ? 0 : 1, 0, ref.data());
                    const double d = rel_diff(got, ref);
                    CHECK(exact ? d == 0.0 : d <= 1e-5, "%s %s %s %dx%d: %g", wn,
                          scheme_name(k).c_str(), boundary_name(b).c_str(), iw, ih, d);
                }
        }
        // transform.cpp:178-196 reference inverse on arbitrary planes
        const Image planes = ref_image(16, 64, 109, exact);
        QuadGrid q(16, 16);
        for (int c = 0; c < 4; ++c)
            q.planes[c].assign(planes.samples.begin() + c * 256, planes.samples.begin() + (c + 1) * 256);
        for (BoundaryMode b : {BoundaryMode::periodic, BoundaryMode::symmetric}) {
            const Image got = inverse(q, w, b, true);
            std::vector<double> ref(32 * 32);
            wlref_inverse(planes.samples.data(), 16, 16, w.id, b == BoundaryMode::periodic ? 0 : 1, 1,
                          ref.data());
            double m = 0;
            for (std::size_t i = 0; i < ref.size(); ++i) m = std::max(m, std::abs(got.samples[i] - ref[i]));
            CHECK(m <= 1e-5 * 4, "inverse %s %s: %g", wn, boundary_name(b).c_str(), m);
        }
    }
    // test_transform.cpp:96-117: impulse through the fused predict (fwd of an
    // impulse equals the reference bit for bit).
    {
        Image img(16, 16);
        img.at(4, 4) = 1.0;
        const QuadGrid got = forward(img, build_scheme(SchemeKind::Monolithic, get_wavelet("cdf53")),
                                     BoundaryMode::periodic, false);
        std::vector<double> ref(256);
        wlref_forward(img.samples.data(), 16, 16, WL_CDF53, 5, 0, 0, ref.data());
        CHECK(rel_diff(got, ref) == 0.0, "impulse");
    }
    // test_transform.cpp:273-305: pyramid shapes + reconstruction
    {
        const WaveletSpec w = get_wavelet("cdf53");
        const Image img = ref_image(64, 32, 110, true);
        const Pyramid p = multi_level_forward(img, build_scheme(SchemeKind::Sweldens, w), 3,
                                              BoundaryMode::periodic, false);
        CHECK(p.details.size() == 3 && p.details[0].w == 32 && p.details[0].h == 16 &&
                  p.details[2].w == 8 && p.details[2].h == 4 && p.ll_w == 8 && p.ll_h == 4 &&
                  p.ll.size() == 32,
              "pyramid shapes");
        const Image rec = multi_level_inverse(p, w, BoundaryMode::periodic, false);
        double m = 0;
        for (std::size_t i = 0; i < rec.samples.size(); ++i)
            m = std::max(m, std::abs(rec.samples[i] - img.samples[i]));
        CHECK(m <= 1e-6, "pyramid roundtrip %g", m);
    }
    // test_transform.cpp:119-125, 307-326: validation errors
    {
        const Scheme s = build_scheme(SchemeKind::Sweldens, get_wavelet("cdf53"));
        bool threw = false;
        try { forward(Image(6, 5), s, BoundaryMode::periodic, false); } catch (const std::invalid_argument&) { threw = true; }
        CHECK(threw, "odd dims");
        threw = false;
        try { multi_level_forward(Image(12, 16), s, 3, BoundaryMode::periodic, false); } catch (const std::invalid_argument&) { threw = true; }
        CHECK(threw, "levels divisibility");
        threw = false;
        try { get_wavelet("haar"); } catch (const std::invalid_argument&) { threw = true; }
        CHECK(threw, "unknown wavelet");
        CHECK(count_barriers(build_scheme(SchemeKind::MonolithicStar, get_wavelet("cdf97"))) == 4 &&
                  count_macs(build_scheme(SchemeKind::MonolithicStar, get_wavelet("cdf97"))) == 36,
              "cost table");
        CHECK(resolve_index(-1, 4, BoundaryMode::symmetric) == 1 &&
                  resolve_index(-1, 4, BoundaryMode::periodic) == 3,
              "resolve_index");
    }
    std::printf("%d checks, %d failures\n", g_checks, g_fail);
    return g_fail ? 1 : 0;
}
