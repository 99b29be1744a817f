// C++ parity test of the drop-in API (include/wavelift_b200.hpp) against the
// UNMODIFIED reference library (oracle/_ref/libwavelift_ref.so, C-ABI of
// oracle/ref_capi.cpp), modelled on proj/tests/test_transform.cpp.
// Built and run by tests/test_cpp_dropin.py on a GPU box. Exit 0 = all pass.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <random>
#include <stdexcept>
#include <vector>

#include "wavelift_b200.hpp"

extern "C" {
long wlref_dump_scheme(int, int, char*, long);
int wlref_apply_step(const double*, int, int, const int*, const double*, int, int, double*);
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
    // schemes.hpp:34-45: walk Scheme::steps like parsim.cpp:250,285-286 does --
    // labels, needs_barrier flags and term counts equal the reference's
    // build_scheme (its JSON dump, oracle/ref_capi.cpp), and every step run
    // through apply_step equals the reference's apply_step on the same planes.
    {
        static const char* wn[] = {"cdf53", "cdf97", "dd137"};
        for (int wi = 0; wi < 3; ++wi)
            for (SchemeKind k : all_scheme_kinds()) {
                const Scheme s = build_scheme(k, get_wavelet(wn[wi]));
                const long len = wlref_dump_scheme(wi, static_cast<int>(k), nullptr, 0);
                std::string js(static_cast<std::size_t>(len) + 1, '\0');
                wlref_dump_scheme(wi, static_cast<int>(k), js.data(), len + 1);
                std::size_t pos = 0;
                int nref = 0;
                for (const Step& st : s.steps) {
                    const std::size_t lp = js.find("\"label\":\"", pos);
                    CHECK(lp != std::string::npos, "%s/%s: fewer reference steps", wn[wi],
                          scheme_name(k).c_str());
                    if (lp == std::string::npos) break;
                    const std::size_t l0 = lp + 9, l1 = js.find('"', l0);
                    const std::string label = js.substr(l0, l1 - l0);
                    const std::size_t bp = js.find("\"barrier\":", l1);
                    const bool barrier = js[bp + 10] == '1';
                    CHECK(label == st.label && barrier == st.needs_barrier &&
                              barrier == st.matrix.needs_barrier(),
                          "%s/%s step %d: %s/%d vs reference %s/%d", wn[wi],
                          scheme_name(k).c_str(), nref, st.label.c_str(), st.needs_barrier,
                          label.c_str(), barrier);
                    pos = l1;
                    ++nref;
                }
                CHECK(js.find("\"label\":\"", pos) == std::string::npos, "%s/%s: extra steps",
                      wn[wi], scheme_name(k).c_str());
                CHECK(k == SchemeKind::Convolution ? (s.steps.empty() && s.conv_filters &&
                                                      s.conv_filters->f_ll.tap_count() > 0)
                                                   : !s.conv_filters.has_value(),
                      "conv filters");
            }
        // apply_step (transform.cpp:100-125): every Monolithic* / Polyphase step
        const int qw = 40, qh = 26;
        QuadGrid q(qw, qh);
        std::mt19937 rng(7);
        for (auto& p : q.planes)
            for (double& v : p) v = static_cast<double>(rng() % 256) / 256.0;
        std::vector<double> in4(4 * qw * qh);
        for (int c = 0; c < 4; ++c) std::copy(q.planes[c].begin(), q.planes[c].end(), in4.begin() + c * qw * qh);
        for (SchemeKind k : {SchemeKind::MonolithicStar, SchemeKind::Polyphase, SchemeKind::Explosive})
            for (const Step& st : build_scheme(k, get_wavelet("cdf53")).steps)
                for (BoundaryMode b : {BoundaryMode::periodic, BoundaryMode::symmetric}) {
                    std::vector<int> idx;
                    std::vector<double> co;
                    for (int r = 0; r < 4; ++r)
                        for (int c = 0; c < 4; ++c)
                            for (const auto& [e, v] : st.matrix.entry(r, c).terms()) {
                                idx.insert(idx.end(), {r, c, e.first, e.second});
                                co.push_back(v);
                            }
                    std::vector<double> want(4 * qw * qh);
                    CHECK(wlref_apply_step(in4.data(), qw, qh, idx.data(), co.data(),
                                           static_cast<int>(co.size()),
                                           b == BoundaryMode::periodic ? 0 : 1, want.data()) == 0,
                          "reference apply_step");
                    const QuadGrid got = apply_step(q, st.matrix, b);
                    double m = 0;
                    for (int c = 0; c < 4; ++c)
                        for (int i = 0; i < qw * qh; ++i)
                            m = std::max(m, std::abs(got.planes[c][i] - want[c * qw * qh + i]));
                    // cdf53 on 8-bit dyadic planes: exact in float32
                    CHECK(m == 0.0, "apply_step %s %s: %g", st.label.c_str(),
                          boundary_name(b).c_str(), m);
                }
        const Scheme conv = build_scheme(SchemeKind::Convolution, get_wavelet("cdf97"));
        const auto mats = scheme_step_matrices(conv);
        CHECK(mats.size() == 1 && mats[0].entry(LL, LL).tap_count() > 0, "conv polyphase matrix");
    }
    std::printf("%d checks, %d failures\n", g_checks, g_fail);
    return g_fail ? 1 : 0;
}
