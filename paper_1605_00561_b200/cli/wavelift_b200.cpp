// wavelift_b200 -- the reference CLI's data-path subcommands on the B200 path
// (proj/tools/wavelift_main.cpp:153-272): `transform` (PGM -> subband
// container), `roundtrip` (forward + inverse, max error) and `bench` (forward
// timing on the reference's mt19937(12345) image). Same options, output lines
// and exit codes (0 ok, 1 usage / invalid argument, 2 failure); the transforms
// run through the drop-in API (include/wavelift_b200.hpp) on the GPU.
// verify / report / simulate are the reference's algebra and simulator tools
// and are not on the data path.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

#include "wavelift_b200.hpp"
#include "wavelift_b200_io.hpp"

using namespace wavelift;

namespace {

constexpr int kExitOk = 0, kExitUsage = 1, kExitFailure = 2;

struct Args {
    std::vector<std::string> pos;
    std::string wavelet = "cdf53", scheme = "sweldens", boundary = "periodic";
    std::string size = "1024x1024", format = "text";
    int levels = 1, reps = 5;
    bool scaling = false, pad = false;
    // opt-in extensions (off: the reference's exact behaviour and output)
    bool scheme_inverse = false;  // roundtrip: the scheme's own inverse kernel
    bool gpix = false;            // bench: add GPix/s to the output
};

int to_int(const std::string& s, const char* what) {
    try {
        std::size_t used = 0;
        const int v = std::stoi(s, &used);
        if (used == s.size()) return v;
    } catch (...) {
    }
    throw std::invalid_argument(std::string("bad ") + what + ": " + s);
}

Args parse(int argc, char** argv, int first) {
    Args a;
    for (int i = first; i < argc; ++i) {
        const std::string k = argv[i];
        auto val = [&]() -> std::string {
            if (i + 1 >= argc) throw std::invalid_argument("missing value for " + k);
            return argv[++i];
        };
        if (k == "--wavelet") a.wavelet = val();
        else if (k == "--scheme") a.scheme = val();
        else if (k == "--boundary") a.boundary = val();
        else if (k == "--levels") a.levels = to_int(val(), "levels");
        else if (k == "--reps") a.reps = to_int(val(), "reps");
        else if (k == "--size") a.size = val();
        else if (k == "--format") a.format = val();
        else if (k == "--scaling") a.scaling = true;
        else if (k == "--pad") a.pad = true;
        else if (k == "--scheme-inverse") a.scheme_inverse = true;
        else if (k == "--gpix") a.gpix = true;
        else if (!k.empty() && k[0] == '-') throw std::invalid_argument("unknown option " + k);
        else a.pos.push_back(k);
    }
    return a;
}

SchemeKind scheme_or_throw(const std::string& name) {
    const auto k = parse_scheme(name);
    if (!k) throw std::invalid_argument("unknown scheme: " + name);
    return *k;
}

BoundaryMode boundary_or_throw(const std::string& name) {
    const auto m = parse_boundary(name);
    if (!m) throw std::invalid_argument("unknown boundary mode: " + name);
    return *m;
}

// wavelift_main.cpp:64-81: odd dimensions need --pad (one mirrored row/col).
Image load_even_image(const std::string& path, bool pad) {
    const Image img = to_image(read_pgm(path));
    if (img.width % 2 == 0 && img.height % 2 == 0) return img;
    if (!pad)
        throw std::invalid_argument("image dimensions are odd (" + std::to_string(img.width) + "x" +
                                    std::to_string(img.height) +
                                    "); rerun with --pad or supply even dimensions");
    const int w = img.width + img.width % 2, h = img.height + img.height % 2;
    Image out(w, h);
    for (int r = 0; r < h; ++r)
        for (int c = 0; c < w; ++c)
            out.at(r, c) = img.at(resolve_index(r, img.height, BoundaryMode::symmetric),
                                  resolve_index(c, img.width, BoundaryMode::symmetric));
    return out;
}

void check_divisible(const Image& img, int levels) {
    if (levels < 1) throw std::invalid_argument("levels must be >= 1");
    const int div = 1 << std::min(levels, 30);
    if (img.width % div != 0 || img.height % div != 0)
        throw std::invalid_argument("image dimensions " + std::to_string(img.width) + "x" +
                                    std::to_string(img.height) + " are not divisible by 2^" +
                                    std::to_string(levels));
}

int cmd_transform(const Args& a) {
    if (a.pos.size() != 2) throw std::invalid_argument("transform needs INPUT and OUTPUT");
    const WaveletSpec w = get_wavelet(a.wavelet);
    const SchemeKind kind = scheme_or_throw(a.scheme);
    const BoundaryMode b = boundary_or_throw(a.boundary);
    const Image img = load_even_image(a.pos[0], a.pad);
    check_divisible(img, a.levels);
    const Pyramid p = multi_level_forward(img, build_scheme(kind, w), a.levels, b, a.scaling);
    SubbandHeader h;
    h.wavelet = w.name;
    h.scheme = scheme_name(kind);
    h.levels = a.levels;
    h.boundary = b;
    h.scaling = a.scaling;
    h.image_w = img.width;
    h.image_h = img.height;
    write_subbands(a.pos[1], h, p);
    std::printf("wrote %s: %d level(s), coarsest %dx%d, %s/%s, %s boundary\n", a.pos[1].c_str(),
                a.levels, p.ll_w, p.ll_h, w.name.c_str(), scheme_name(kind).c_str(),
                boundary_name(b).c_str());
    return kExitOk;
}

int cmd_roundtrip(const Args& a) {
    if (a.pos.size() != 1) throw std::invalid_argument("roundtrip needs INPUT");
    const WaveletSpec w = get_wavelet(a.wavelet);
    const SchemeKind kind = scheme_or_throw(a.scheme);
    const BoundaryMode b = boundary_or_throw(a.boundary);
    const Image img = load_even_image(a.pos[0], false);
    check_divisible(img, a.levels);
    if (b == BoundaryMode::symmetric && kind != SchemeKind::Sweldens)
        std::fprintf(stderr,
                     "note: %s under the symmetric boundary matches the separable "
                     "factorization only away from image borders; reconstruction is "
                     "exact for --scheme sweldens or --boundary periodic\n",
                     scheme_name(kind).c_str());
    const Pyramid p = multi_level_forward(img, build_scheme(kind, w), a.levels, b, false);
    // The reference always inverts with the wavelet-only (Sweldens) inverse
    // (wavelift_main.cpp:196); --scheme-inverse runs the scheme's own kernel.
    const Image rec = a.scheme_inverse ? multi_level_inverse(p, w, b, false, kind)
                                       : multi_level_inverse(p, w, b, false);
    double err = 0.0;
    for (std::size_t i = 0; i < img.samples.size(); ++i)
        err = std::max(err, std::abs(img.samples[i] - rec.samples[i]));
    // float32 arithmetic: the reference's 1e-6 (float64) becomes 3e-5
    // (the bound the GPU perfect-reconstruction tests use)
    const double tol = 3e-5;
    const bool ok = err <= tol;
    std::printf("roundtrip %s/%s levels=%d %s: max abs error %.3g (tolerance %g) %s\n",
                w.name.c_str(), scheme_name(kind).c_str(), a.levels, boundary_name(b).c_str(), err,
                tol, ok ? "OK" : "FAIL");
    return ok ? kExitOk : kExitFailure;
}

int cmd_bench(const Args& a) {
    if (a.reps < 1) throw std::invalid_argument("reps must be >= 1");
    const WaveletSpec w = get_wavelet(a.wavelet);
    const SchemeKind kind = scheme_or_throw(a.scheme);
    const auto x = a.size.find('x');
    int bw = 0, bh = 0;
    if (x != std::string::npos) {
        bw = to_int(a.size.substr(0, x), "size");
        bh = to_int(a.size.substr(x + 1), "size");
    }
    if (bw <= 0 || bh <= 0) throw std::invalid_argument("bad size '" + a.size + "', expected WxH");
    if (bw % 2 || bh % 2) throw std::invalid_argument("bench size must have even dimensions");
    // the reference's input: mt19937(12345) uniform [0, 1) (wavelift_main.cpp:245-248)
    std::vector<float> host(static_cast<std::size_t>(bw) * bh);
    std::mt19937 rng(12345);
    std::uniform_real_distribution<double> dist(0.0, 1.0);
    for (float& v : host) v = static_cast<float>(dist(rng));
    const std::size_t n = static_cast<std::size_t>(bw / 2) * (bh / 2);
    float *d_img = nullptr, *d_q = nullptr;
    if (cudaMalloc(&d_img, host.size() * 4) != cudaSuccess || cudaMalloc(&d_q, 4 * n * 4) != cudaSuccess)
        throw std::runtime_error("cudaMalloc failed");
    cudaMemcpy(d_img, host.data(), host.size() * 4, cudaMemcpyHostToDevice);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto run = [&]() {
        const int st = wl_dwt2_forward(d_img, bw, bh, bw, w.id, static_cast<int>(kind), WL_PERIODIC,
                                       0, d_q, d_q + n, d_q + 2 * n, d_q + 3 * n, bw / 2, nullptr);
        if (st != WL_OK) throw std::runtime_error(wl_last_error());
    };
    run();
    std::vector<double> seconds;
    for (int r = 0; r < a.reps; ++r) {
        cudaEventRecord(e0);
        run();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        seconds.push_back(ms * 1e-3);
    }
    float ll00 = 0.f;
    cudaMemcpy(&ll00, d_q, 4, cudaMemcpyDeviceToHost);
    cudaFree(d_img);
    cudaFree(d_q);
    if (!std::isfinite(ll00)) return kExitFailure;
    std::sort(seconds.begin(), seconds.end());
    const std::size_t m = seconds.size();
    const double med = (seconds[(m - 1) / 2] + seconds[m / 2]) / 2.0;
    const double mbps = static_cast<double>(bw) * bh * 8.0 / med / 1e6;  // the reference's unit
    const double gpix = static_cast<double>(bw) * bh / med / 1e9;
    // wavelift_main.cpp:264-269 output; --gpix appends the GPixel/s figure
    if (a.format == "csv" && a.gpix)
        std::printf("scheme,wavelet,size,mbps,gpix_s\n%s,%s,%dx%d,%.2f,%.2f\n",
                    scheme_name(kind).c_str(), w.name.c_str(), bw, bh, mbps, gpix);
    else if (a.format == "csv")
        std::printf("scheme,wavelet,size,mbps\n%s,%s,%dx%d,%.2f\n", scheme_name(kind).c_str(),
                    w.name.c_str(), bw, bh, mbps);
    else if (a.gpix)
        std::printf("%s/%s %dx%d: median %.2f MB/s over %d rep(s) (%.1f GPix/s, B200 float32)\n",
                    scheme_name(kind).c_str(), w.name.c_str(), bw, bh, mbps, a.reps, gpix);
    else
        std::printf("%s/%s %dx%d: median %.2f MB/s over %d rep(s)\n", scheme_name(kind).c_str(),
                    w.name.c_str(), bw, bh, mbps, a.reps);
    return kExitOk;
}

void usage() {
    std::fprintf(stderr,
                 "usage: wavelift_b200 transform INPUT OUTPUT [--wavelet W] [--scheme S] "
                 "[--levels L] [--boundary B] [--scaling] [--pad]\n"
                 "       wavelift_b200 roundtrip INPUT [--wavelet W] [--scheme S] [--levels L] "
                 "[--boundary B] [--scheme-inverse]\n"
                 "       wavelift_b200 bench [--size WxH] [--wavelet W] [--scheme S] [--reps N] "
                 "[--format text|csv] [--gpix]\n");
}

}  // namespace

int main(int argc, char** argv) {
    if (argc < 2) {
        usage();
        return kExitUsage;
    }
    const std::string cmd = argv[1];
    try {
        const Args a = parse(argc, argv, 2);
        if (cmd == "transform") return cmd_transform(a);
        if (cmd == "roundtrip") return cmd_roundtrip(a);
        if (cmd == "bench") return cmd_bench(a);
        usage();
        return kExitUsage;
    } catch (const std::invalid_argument& e) {  // wavelift_main.cpp:363-369
        std::fprintf(stderr, "error: %s\n", e.what());
        return kExitUsage;
    } catch (const std::exception& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return kExitFailure;
    }
}
