// C-ABI entry points (include/wl_dwt.h): argument validation with the
// reference's error semantics, engine dispatch, and the multi-level pyramid
// driver (transform.cpp:198-256).
#include <atomic>
#include <cstdio>
#include <cstring>
#include <string>

#include "../../include/wl_dwt.h"
#include "wl_internal.h"

namespace {

thread_local std::string g_err;
std::atomic<long> g_launches{0};
std::atomic<int> g_engine{0};

int fail(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

int cuda_status(cudaError_t e, const char* where) {
    if (e == cudaSuccess) return WL_OK;
    return fail(WL_ERUNTIME, std::string(where) + ": " + cudaGetErrorString(e));
}

bool valid_ids(int wavelet, int scheme, int boundary) {
    return wavelet >= 0 && wavelet <= 2 && scheme >= 0 && scheme <= 9 && boundary >= 0 &&
           boundary <= 1;
}

int prog_index(int wavelet, int scheme, int direction) {
    return (wavelet * 10 + scheme) * 2 + direction;
}

// Single-level launch with engine selection.
int launch_level(WlLevel L, cudaStream_t s) {
    if (L.direction == 1 && L.scheme == WL_CONVOLUTION) {
        L.scheme = WL_SWELDENS;  // no lifting factorisation: reference inverse
        L.prog = prog_index(L.wavelet, L.scheme, 1);
    }
    const WlProgram& P = wl_host_program(L.prog);
    cudaError_t e;
    const int engine = g_engine.load();
    if (P.is_conv) {
        e = (engine != 1 && L.wavelet <= 1) ? wl_launch_conv_fast(L, s) : wl_launch_conv(L, s);
        return cuda_status(e, "conv_kernel");
    }
    if (engine == 2 && !wl_fast_supported(L))
        return fail(WL_EINVAL, "fast engine does not support this wavelet/scheme");
    if (engine != 1 && wl_fast_supported(L)) {
        e = wl_launch_fast(L, s);
        return cuda_status(e, "fast_kernel");
    }
    e = wl_launch_interp(L, s);
    return cuda_status(e, "interp_kernel");
}

}  // namespace

void wl_count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

extern "C" {

const char* wl_last_error(void) { return g_err.c_str(); }

const char* wl_version(void) {
    return "wavelift_b200 0.1 (sm_100a; generic tile interpreter + fast register-tile engine)";
}

int wl_set_engine(int engine) { return g_engine.exchange(engine); }

long wl_launch_count(void) { return g_launches.load(); }

int wl_resolve_index(int i, int n, int boundary) {
    // transform.cpp:59-72
    if (i >= 0 && i < n) return i;
    if (n == 1) return 0;
    if (boundary == WL_PERIODIC) {
        int m = i % n;
        return m < 0 ? m + n : m;
    }
    while (i < 0 || i >= n) {
        if (i < 0) i = -i;
        if (i >= n) i = 2 * (n - 1) - i;
    }
    return i;
}

int wl_scheme_info(int wavelet, int scheme, int direction, int* barriers, long* macs,
                   int* epochs, int* halo) {
    if (!valid_ids(wavelet, scheme, 0) || direction < 0 || direction > 1)
        return fail(WL_EINVAL, "unknown wavelet/scheme/direction");
    if (direction == 1 && scheme == WL_CONVOLUTION) scheme = WL_SWELDENS;
    const WlProgram& P = wl_host_program(prog_index(wavelet, scheme, direction));
    if (barriers) *barriers = P.barriers;
    if (macs) *macs = P.macs;
    if (epochs) *epochs = P.is_conv ? 1 : P.nbr_steps;
    if (halo) *halo = P.is_conv ? (P.creach + 1) / 2 : P.halo;
    return WL_OK;
}

int wl_dwt2_forward(const float* img, int w, int h, long img_pitch, int wavelet, int scheme,
                    int boundary, int scaling, float* ll, float* hl, float* lh, float* hh,
                    long plane_pitch, void* stream) {
    // transform.cpp:165-166: even positive dimensions or invalid_argument.
    if (w <= 0 || h <= 0 || w % 2 != 0 || h % 2 != 0)
        return fail(WL_EINVAL, "forward requires even positive dimensions");
    if (!valid_ids(wavelet, scheme, boundary))
        return fail(WL_EINVAL, "unknown wavelet/scheme/boundary");
    if (!img || !ll || !hl || !lh || !hh) return fail(WL_EINVAL, "null buffer");
    if (img_pitch < w || plane_pitch < w / 2) return fail(WL_EINVAL, "pitch too small");
    WlLevel L{};
    L.in[0] = img;
    L.out[0] = ll;
    L.out[1] = hl;
    L.out[2] = lh;
    L.out[3] = hh;
    L.qw = w / 2;
    L.qh = h / 2;
    L.in_pitch = img_pitch;
    L.out_pitch = plane_pitch;
    L.wavelet = wavelet;
    L.scheme = scheme;
    L.direction = 0;
    L.prog = prog_index(wavelet, scheme, 0);
    L.boundary = boundary;
    L.scaling = scaling != 0;
    return launch_level(L, static_cast<cudaStream_t>(stream));
}

int wl_dwt2_inverse(const float* ll, const float* hl, const float* lh, const float* hh, int qw,
                    int qh, long plane_pitch, int wavelet, int scheme, int boundary,
                    int undo_scaling, float* img, long img_pitch, void* stream) {
    if (qw <= 0 || qh <= 0) return fail(WL_EINVAL, "inverse requires positive plane dimensions");
    if (!valid_ids(wavelet, scheme, boundary))
        return fail(WL_EINVAL, "unknown wavelet/scheme/boundary");
    if (!img || !ll || !hl || !lh || !hh) return fail(WL_EINVAL, "null buffer");
    if (img_pitch < 2 * qw || plane_pitch < qw) return fail(WL_EINVAL, "pitch too small");
    WlLevel L{};
    L.in[0] = ll;
    L.in[1] = hl;
    L.in[2] = lh;
    L.in[3] = hh;
    L.out[0] = img;
    L.qw = qw;
    L.qh = qh;
    L.in_pitch = plane_pitch;
    L.out_pitch = img_pitch;
    L.wavelet = wavelet;
    L.scheme = scheme;
    L.direction = 1;
    L.prog = prog_index(wavelet, scheme, 1);
    L.boundary = boundary;
    L.scaling = undo_scaling != 0;
    return launch_level(L, static_cast<cudaStream_t>(stream));
}

size_t wl_pyramid_elems(int w, int h, int levels) {
    if (w <= 0 || h <= 0 || levels < 1) return 0;
    return static_cast<size_t>(w) * static_cast<size_t>(h);  // sum of 3n_l + n_L = w*h
}

size_t wl_pyramid_scratch_elems(int w, int h, int levels) {
    if (w <= 0 || h <= 0 || levels < 1) return 0;
    // Two ping-pong LL buffers of the level-1 plane size.
    return 2 * static_cast<size_t>(w / 2) * static_cast<size_t>(h / 2);
}

// transform.cpp:198-227: level l transforms the previous level's LL.
int wl_dwt2_pyramid_forward(const float* img, int w, int h, int levels, int wavelet, int scheme,
                            int boundary, int scaling, float* pyramid, float* scratch,
                            void* stream) {
    if (levels < 1) return fail(WL_EINVAL, "levels must be >= 1");
    if (w <= 0 || h <= 0) return fail(WL_EINVAL, "forward requires even positive dimensions");
    const int div = 1 << levels;
    if (levels > 30 || w % div != 0 || h % div != 0)
        return fail(WL_EINVAL, "image dimensions must be divisible by 2^levels");
    if (!img || !pyramid || !scratch) return fail(WL_EINVAL, "null buffer");
    size_t off = 0;
    const float* src = img;
    long src_pitch = w;
    int cw = w, ch = h;
    float* ping[2] = {scratch, scratch + static_cast<size_t>(w / 2) * (h / 2)};
    for (int l = 0; l < levels; ++l) {
        const int qw = cw / 2, qh = ch / 2;
        const size_t n = static_cast<size_t>(qw) * qh;
        float* hl = pyramid + off;
        float* lh = hl + n;
        float* hh = lh + n;
        off += 3 * n;
        float* ll = (l + 1 == levels) ? pyramid + off : ping[l & 1];
        const int st = wl_dwt2_forward(src, cw, ch, src_pitch, wavelet, scheme, boundary, scaling,
                                       ll, hl, lh, hh, qw, stream);
        if (st != WL_OK) return st;
        src = ll;
        src_pitch = qw;
        cw = qw;
        ch = qh;
    }
    return WL_OK;
}

// transform.cpp:229-256: coarsest level first.
int wl_dwt2_pyramid_inverse(const float* pyramid, int w, int h, int levels, int wavelet,
                            int scheme, int boundary, int undo_scaling, float* img,
                            float* scratch, void* stream) {
    if (levels < 1) return fail(WL_EINVAL, "levels must be >= 1");
    const int div = 1 << (levels > 30 ? 30 : levels);
    if (w <= 0 || h <= 0 || levels > 30 || w % div != 0 || h % div != 0)
        return fail(WL_EINVAL, "pyramid level dimensions are inconsistent");
    if (!img || !pyramid || !scratch) return fail(WL_EINVAL, "null buffer");
    size_t offs[32];
    size_t off = 0;
    for (int l = 0; l < levels; ++l) {
        offs[l] = off;
        off += 3 * static_cast<size_t>(w >> (l + 1)) * (h >> (l + 1));
    }
    const float* ll = pyramid + off;  // coarsest LL
    float* ping[2] = {scratch, scratch + static_cast<size_t>(w / 2) * (h / 2)};
    for (int l = levels - 1; l >= 0; --l) {
        const int qw = w >> (l + 1), qh = h >> (l + 1);
        const size_t n = static_cast<size_t>(qw) * qh;
        const float* hl = pyramid + offs[l];
        float* out = (l == 0) ? img : ping[l & 1];
        const int st = wl_dwt2_inverse(ll, hl, hl + n, hl + 2 * n, qw, qh, qw, wavelet, scheme,
                                       boundary, undo_scaling, out, 2 * qw, stream);
        if (st != WL_OK) return st;
        ll = out;
    }
    return WL_OK;
}

}  // extern "C"
