// File-format parity (CPU only): the B200 drop-in's PGM and subband-container
// code (include/wavelift_b200_io.hpp) against the UNMODIFIED reference
// implementation (proj/src/pgm.cpp, proj/src/subband_io.cpp via
// oracle/ref_capi.cpp): identical bytes written, identical values read back,
// same errors on malformed files (test_io.cpp:40-246 in the reference).
#include <cstdio>
#include <fstream>
#include <iterator>
#include <random>
#include <string>
#include <vector>

#include "wavelift_b200_io.hpp"

extern "C" {
int wlref_write_pgm(const char*, int, int, int, const unsigned short*);
int wlref_read_pgm(const char*, int*, int*, int*, unsigned short*);
int wlref_write_subbands(const char*, const char*, const char*, int, int, int, int, int,
                         const double*);
int wlref_read_subbands(const char*, char*, char*, int*, int*, int*, int*, int*, double*);
}

using namespace wavelift;

static int g_fail = 0;
#define CHECK(c, ...)                                                \
    do {                                                             \
        if (!(c)) {                                                  \
            ++g_fail;                                                \
            std::printf("FAIL %s:%d ", __FILE__, __LINE__);          \
            std::printf(__VA_ARGS__);                                \
            std::printf("\n");                                       \
        }                                                            \
    } while (0)

static std::string slurp(const std::string& p) {
    std::ifstream f(p, std::ios::binary);
    return std::string(std::istreambuf_iterator<char>(f), {});
}

int main(int argc, char** argv) {
    const std::string dir = argc > 1 ? argv[1] : "/tmp";
    std::mt19937 rng(7);
    // ---- PGM 8- and 16-bit, odd sizes, both directions
    for (int maxval : {255, 4095, 65535}) {
        PgmImage p;
        p.width = 13;
        p.height = 7;
        p.maxval = maxval;
        for (int i = 0; i < p.width * p.height; ++i) p.pixels.push_back(rng() % (maxval + 1));
        const std::string a = dir + "/b200.pgm", b = dir + "/ref.pgm";
        write_pgm(a, p);
        CHECK(wlref_write_pgm(b.c_str(), p.width, p.height, maxval, p.pixels.data()) == 0, "ref write");
        CHECK(slurp(a) == slurp(b), "PGM bytes differ (maxval %d)", maxval);
        int w, h, mv;
        std::vector<unsigned short> px(p.pixels.size());
        CHECK(wlref_read_pgm(a.c_str(), &w, &h, &mv, px.data()) == 0, "ref read");
        CHECK(w == 13 && h == 7 && mv == maxval && px == p.pixels, "ref reads ours");
        const PgmImage q = read_pgm(b);
        CHECK(q.pixels == p.pixels && q.maxval == maxval, "we read the reference's");
        const Image img = to_image(q);
        CHECK(img.samples[3] == p.pixels[3] / (maxval + 1.0), "to_image normalisation");
        CHECK(from_image(img, maxval).pixels == p.pixels, "from_image inverts to_image");
    }
    {  // comment lines in the header
        std::ofstream f(dir + "/c.pgm", std::ios::binary);
        f << "P5\n# a comment\n2 2 # trailing\n255\n";
        f.put(1); f.put(2); f.put(3); f.put(4);
    }
    CHECK(read_pgm(dir + "/c.pgm").pixels[3] == 4, "comments in the PGM header");
    // ---- subband container: both writers give identical bytes; cross reads
    for (int levels : {1, 3}) {
        const int W = 32, H = 24;
        std::vector<double> flat(W * H);
        std::uniform_real_distribution<double> u(-2, 2);
        for (double& v : flat) v = u(rng);
        Pyramid p;
        std::size_t off = 0;
        for (int l = 0; l < levels; ++l) {
            PyramidLevel lv;
            lv.w = W >> (l + 1);
            lv.h = H >> (l + 1);
            const std::size_t n = static_cast<std::size_t>(lv.w) * lv.h;
            lv.hl.assign(flat.begin() + off, flat.begin() + off + n);
            lv.lh.assign(flat.begin() + off + n, flat.begin() + off + 2 * n);
            lv.hh.assign(flat.begin() + off + 2 * n, flat.begin() + off + 3 * n);
            off += 3 * n;
            p.details.push_back(lv);
        }
        p.ll_w = W >> levels;
        p.ll_h = H >> levels;
        p.ll.assign(flat.begin() + off, flat.end());
        SubbandHeader hd{"cdf97", "monolithic_star", levels, BoundaryMode::symmetric, true, W, H};
        const std::string a = dir + "/b200.sub", b = dir + "/ref.sub";
        write_subbands(a, hd, p);
        CHECK(wlref_write_subbands(b.c_str(), "cdf97", "monolithic_star", levels, 1, 1, W, H,
                                   flat.data()) == 0, "ref write_subbands");
        CHECK(slurp(a) == slurp(b), "subband file bytes differ (levels %d)", levels);
        char wv[64], sc[64];
        int lv, bd, scl, w, h;
        std::vector<double> back(W * H);
        CHECK(wlref_read_subbands(a.c_str(), wv, sc, &lv, &bd, &scl, &w, &h, back.data()) == 0,
              "ref read_subbands");
        CHECK(back == flat && lv == levels && bd == 1 && scl == 1 && w == W && h == H &&
                  std::string(wv) == "cdf97" && std::string(sc) == "monolithic_star",
              "reference reads ours");
        const auto [h2, p2] = read_subbands(b);
        CHECK(h2.levels == levels && h2.scheme == "monolithic_star" && p2.ll == p.ll &&
                  p2.details.back().hh == p.details.back().hh,
              "we read the reference's");
        // truncated payload -> runtime_error, like the reference
        const std::string bytes = slurp(a);
        std::ofstream(dir + "/t.sub", std::ios::binary) << bytes.substr(0, bytes.size() - 8);
        bool threw = false;
        try {
            read_subbands(dir + "/t.sub");
        } catch (const std::runtime_error&) {
            threw = true;
        }
        CHECK(threw, "truncated payload must throw");
        CHECK(wlref_read_subbands((dir + "/t.sub").c_str(), wv, sc, &lv, &bd, &scl, &w, &h,
                                  back.data()) == 2, "reference rejects it too");
    }
    std::printf("%s: %d failure(s)\n", g_fail ? "FAIL" : "PASS", g_fail);
    return g_fail ? 1 : 0;
}
