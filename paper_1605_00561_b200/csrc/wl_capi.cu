// C-ABI entry points (include/wl_dwt.h): argument validation with the
// reference's error semantics, engine dispatch, and the multi-level pyramid
// driver (transform.cpp:198-256).
#include <atomic>
#include <cstdint>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

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
    if ((engine == 2 || engine == 3) && !wl_fast_supported(L))
        return fail(WL_EINVAL, "fast engine does not support this wavelet/scheme");
    if (engine != 1 && wl_fast_supported(L)) {
        e = wl_launch_fast(L, s);
        return cuda_status(e, "fast_kernel");
    }
    e = wl_launch_interp(L, s);
    return cuda_status(e, "interp_kernel");
}

// Batched launch: the fast engine / conv kernel take the batch in one launch
// (3-D TMA maps); every other engine loops over the images.
int launch_level_batch(WlLevel L, cudaStream_t s) {
    if (L.nb <= 1) {
        L.nb = 1;
        return launch_level(L, s);
    }
    WlLevel Lp = L;
    if (Lp.direction == 1 && Lp.scheme == WL_CONVOLUTION) {
        Lp.scheme = WL_SWELDENS;
        Lp.prog = prog_index(Lp.wavelet, Lp.scheme, 1);
    }
    const WlProgram& P = wl_host_program(Lp.prog);
    const int engine = g_engine.load();
    const bool batched = engine != 1 && (P.is_conv ? (Lp.wavelet <= 1 && L.in_bstride[0] % 4 == 0)
                                                   : wl_fast_supported(Lp));
    if (batched) return launch_level(L, s);
    for (int b = 0; b < L.nb; ++b) {
        WlLevel Li = L;
        Li.nb = 1;
        for (int k = 0; k < 4; ++k) {
            if (Li.in[k]) Li.in[k] += b * L.in_bstride[k];
            if (Li.out[k]) Li.out[k] += b * L.out_bstride[k];
        }
        const int st = launch_level(Li, s);
        if (st != WL_OK) return st;
    }
    return WL_OK;
}

// Strip halo in pixel rows (forward) / plane rows (inverse) the fast engine
// needs around a window: the program's reach plus the tiles' ghost row.
int strip_halo(int wavelet, int direction) {
    const int H = wavelet == WL_CDF53 ? 1 : 2;  // required_halo (parsim.cpp:185-218)
    return direction == 0 ? 2 * (H + 1) : H + 1;
}

}  // namespace

void wl_count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

static unsigned long long* g_diag = nullptr;
unsigned long long* wl_diag_ptr() { return g_diag; }

int wl_engine() { return g_engine.load(); }

int wl_fail(int code, const char* msg) { return fail(code, msg); }

extern "C" {

const char* wl_last_error(void) { return g_err.c_str(); }

const char* wl_version(void) {
    return "wavelift_b200 0.1 (sm_100a; generic tile interpreter + fast register-tile engine)";
}

int wl_set_engine(int engine) { return g_engine.exchange(engine); }


long wl_launch_count(void) { return g_launches.load(); }

// Tuning diagnostics: a device buffer of 4 x grid u64 that WL_DIAG_TIMES
// builds of the fast engine fill per CTA (entry, first tile ready, exit,
// tiles processed; %globaltimer ns). Null disables. Not part of the drop-in.
void wl_diag_set(void* dev_buf) { g_diag = static_cast<unsigned long long*>(dev_buf); }

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

int wl_dwt2_forward_batch(const float* img, int w, int h, long img_pitch, long img_stride,
                          int n, int wavelet, int scheme, int boundary, int scaling, float* ll,
                          float* hl, float* lh, float* hh, long plane_pitch, long plane_stride,
                          void* stream) {
    if (n < 0) return fail(WL_EINVAL, "batch size must be >= 0");
    if (n == 0) return WL_OK;
    if (w <= 0 || h <= 0 || w % 2 != 0 || h % 2 != 0)
        return fail(WL_EINVAL, "forward requires even positive dimensions");
    if (!valid_ids(wavelet, scheme, boundary))
        return fail(WL_EINVAL, "unknown wavelet/scheme/boundary");
    if (!img || !ll || !hl || !lh || !hh) return fail(WL_EINVAL, "null buffer");
    if (img_pitch < w || plane_pitch < w / 2) return fail(WL_EINVAL, "pitch too small");
    if (n > 1 && (img_stride < img_pitch * h || plane_stride < plane_pitch * (h / 2)))
        return fail(WL_EINVAL, "batch stride too small");
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
    L.nb = n;
    L.in_bstride[0] = img_stride;
    for (int k = 0; k < 4; ++k) L.out_bstride[k] = plane_stride;
    return launch_level_batch(L, static_cast<cudaStream_t>(stream));
}

int wl_dwt2_inverse_batch(const float* ll, const float* hl, const float* lh, const float* hh,
                          int qw, int qh, long plane_pitch, long plane_stride, int n, int wavelet,
                          int scheme, int boundary, int undo_scaling, float* img, long img_pitch,
                          long img_stride, void* stream) {
    if (n < 0) return fail(WL_EINVAL, "batch size must be >= 0");
    if (n == 0) return WL_OK;
    if (qw <= 0 || qh <= 0) return fail(WL_EINVAL, "inverse requires positive plane dimensions");
    if (!valid_ids(wavelet, scheme, boundary))
        return fail(WL_EINVAL, "unknown wavelet/scheme/boundary");
    if (!img || !ll || !hl || !lh || !hh) return fail(WL_EINVAL, "null buffer");
    if (img_pitch < 2 * qw || plane_pitch < qw) return fail(WL_EINVAL, "pitch too small");
    if (n > 1 && (img_stride < img_pitch * 2 * qh || plane_stride < plane_pitch * qh))
        return fail(WL_EINVAL, "batch stride too small");
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
    L.nb = n;
    for (int k = 0; k < 4; ++k) L.in_bstride[k] = plane_stride;
    L.out_bstride[0] = img_stride;
    return launch_level_batch(L, static_cast<cudaStream_t>(stream));
}

int wl_strip_halo_rows(int wavelet, int scheme, int direction) {
    if (!valid_ids(wavelet, scheme, 0) || wavelet > WL_CDF97 || direction < 0 || direction > 1)
        return -1;
    return strip_halo(wavelet, direction);
}

int wl_dwt2_forward_strip(const float* strip, int w, int rows, int halo_rows, long pitch,
                          int wavelet, int scheme, int scaling, float* ll, float* hl, float* lh,
                          float* hh, long plane_pitch, void* stream) {
    return wl_forward_strip_wait(strip, w, rows, halo_rows, pitch, wavelet, scheme, scaling, ll,
                                 hl, lh, hh, plane_pitch, stream, nullptr, nullptr, 0, nullptr,
                                 WL_PERIODIC, -1, -1);
}

}  // extern "C"

bool wl_strip_wait_capable(int wavelet, int scheme) {
    return !wl_host_program(prog_index(wavelet, scheme, 0)).is_conv;
}

static bool P_is_conv(int wavelet, int scheme) {
    return wl_host_program(prog_index(wavelet, scheme, 0)).is_conv;
}

int wl_forward_strip_wait(const float* strip, int w, int rows, int halo_rows, long pitch,
                          int wavelet, int scheme, int scaling, float* ll, float* hl, float* lh,
                          float* hh, long plane_pitch, void* stream, const unsigned* xflag_a,
                          const unsigned* xflag_b, unsigned xepoch, unsigned* xerr,
                          int boundary, int halo_top, int halo_bot) {
    if (w <= 0 || rows <= 0 || w % 2 != 0 || rows % 2 != 0)
        return fail(WL_EINVAL, "forward requires even positive dimensions");
    if (!valid_ids(wavelet, scheme, 0) || wavelet > WL_CDF97)
        return fail(WL_EINVAL, "strip transforms support cdf53/cdf97");
    if (halo_top < 0) halo_top = halo_rows;
    if (halo_bot < 0) halo_bot = halo_rows;
    // periodic windows read a halo on both sides; a symmetric window may sit
    // on the image's own top/bottom edge (halo 0 there: mirrored, exact)
    const bool sym = boundary == WL_SYMMETRIC;
    for (int hr : {halo_top, halo_bot})
        if (hr % 2 != 0 || (hr < strip_halo(wavelet, 0) && !(sym && hr == 0)))
            return fail(WL_EINVAL, "strip halo too small (see wl_strip_halo_rows) or odd");
    if (!strip || !ll || !hl || !lh || !hh) return fail(WL_EINVAL, "null buffer");
    if (pitch < w || plane_pitch < w / 2) return fail(WL_EINVAL, "pitch too small");
    if (P_is_conv(wavelet, scheme) && sym)
        return fail(WL_EINVAL, "symmetric strips need a lifting scheme");
    WlLevel L{};
    L.in[0] = strip - static_cast<long>(halo_top) * pitch;
    L.out[0] = ll;
    L.out[1] = hl;
    L.out[2] = lh;
    L.out[3] = hh;
    L.qw = w / 2;
    L.qh = rows / 2 + (halo_top + halo_bot) / 2;
    L.in_pitch = pitch;
    L.out_pitch = plane_pitch;
    L.wavelet = wavelet;
    L.scheme = scheme;
    L.direction = 0;
    L.prog = prog_index(wavelet, scheme, 0);
    L.boundary = sym ? WL_SYMMETRIC : WL_PERIODIC;
    L.scaling = scaling != 0;
    L.ylo = halo_top / 2;
    L.yhi = L.ylo + rows / 2;
    L.xflag_a = xflag_a;
    L.xflag_b = xflag_b;
    L.xepoch = xepoch;
    L.xerr = xerr;
    const WlProgram& P = wl_host_program(L.prog);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (P.is_conv) {
        if (xflag_a) return fail(WL_EINVAL, "halo wait needs a lifting scheme");
        return cuda_status(wl_launch_conv_fast(L, s), "conv_kernel");
    }
    if (!wl_fast_supported(L))
        return fail(WL_EINVAL, "strip transform needs 16-byte aligned buffers and pitches");
    return cuda_status(wl_launch_fast(L, s), "fast_kernel");
}

bool wl_strip_shape_ok(int w, int rows, int halo_rows, int wavelet, int scheme, int direction) {
    return wl_strip_mode(w, rows, halo_rows, wavelet, scheme, direction) != 0;
}

int wl_strip_mode(int w, int rows, int halo_rows, int wavelet, int scheme, int direction) {
    return wl_strip_mode_b(w, rows, halo_rows, halo_rows, wavelet, scheme, direction, WL_PERIODIC);
}

int wl_strip_mode_b(int w, int rows, int halo_top, int halo_bot, int wavelet, int scheme,
                    int direction, int boundary) {
    const int halo_rows = halo_top;
    if (w <= 0 || rows <= 0 || !valid_ids(wavelet, scheme, 0) || wavelet > WL_CDF97) return 0;
    if (direction == 1 && scheme == WL_CONVOLUTION) scheme = WL_SWELDENS;
    const WlProgram& P = wl_host_program(prog_index(wavelet, scheme, direction));
    if (P.is_conv) {
        if (boundary == WL_SYMMETRIC) return 0;
        return w % 2 == 0 && rows % 2 == 0 ? 3 : 0;  // any even shape
    }
    // a level descriptor shaped like the strip call's, at dummy aligned addresses
    const float* dummy = reinterpret_cast<const float*>(static_cast<uintptr_t>(1) << 20);
    WlLevel L{};
    L.wavelet = wavelet;
    L.scheme = scheme;
    L.direction = direction;
    L.prog = prog_index(wavelet, scheme, direction);
    L.boundary = boundary;
    for (int k = 0; k < 4; ++k) {
        L.in[k] = dummy;
        L.out[k] = const_cast<float*>(dummy);
    }
    if (direction == 0) {
        if (w % 2 || rows % 2 || halo_top % 2 || halo_bot % 2) return 0;
        L.qw = w / 2;
        L.qh = rows / 2 + (halo_top + halo_bot) / 2;
        L.in_pitch = w;
        L.out_pitch = w / 2;
        L.ylo = halo_top / 2;
        L.yhi = L.ylo + rows / 2;
    } else {
        L.qw = w;
        L.qh = rows + halo_top + halo_bot;
        L.in_pitch = w;
        L.out_pitch = 2 * w;
        L.ylo = halo_top;
        L.yhi = halo_top + rows;
    }
    (void)halo_rows;
    return wl_fast_mode(L);
}

int wl_inverse_strip_ex(const float* ll, const float* hl, const float* lh, const float* hh,
                        int qw, int qrows, int halo_top, int halo_bot, long plane_pitch,
                        int wavelet, int scheme, int undo_scaling, float* img, long img_pitch,
                        void* stream, int boundary) {
    if (qw <= 0 || qrows <= 0) return fail(WL_EINVAL, "inverse requires positive plane dimensions");
    if (!valid_ids(wavelet, scheme, 0) || wavelet > WL_CDF97)
        return fail(WL_EINVAL, "strip transforms support cdf53/cdf97");
    const bool sym = boundary == WL_SYMMETRIC;
    for (int hr : {halo_top, halo_bot})
        if (hr < strip_halo(wavelet, 1) && !(sym && hr == 0))
            return fail(WL_EINVAL, "strip halo too small (see wl_strip_halo_rows)");
    if (!img || !ll || !hl || !lh || !hh) return fail(WL_EINVAL, "null buffer");
    if (img_pitch < 2 * qw || plane_pitch < qw) return fail(WL_EINVAL, "pitch too small");
    if (scheme == WL_CONVOLUTION) scheme = WL_SWELDENS;
    const long back = static_cast<long>(halo_top) * plane_pitch;
    WlLevel L{};
    L.in[0] = ll - back;
    L.in[1] = hl - back;
    L.in[2] = lh - back;
    L.in[3] = hh - back;
    L.out[0] = img;
    L.qw = qw;
    L.qh = qrows + halo_top + halo_bot;
    L.in_pitch = plane_pitch;
    L.out_pitch = img_pitch;
    L.wavelet = wavelet;
    L.scheme = scheme;
    L.direction = 1;
    L.prog = prog_index(wavelet, scheme, 1);
    L.boundary = sym ? WL_SYMMETRIC : WL_PERIODIC;
    L.scaling = undo_scaling != 0;
    L.ylo = halo_top;
    L.yhi = halo_top + qrows;
    if (!wl_fast_supported(L))
        return fail(WL_EINVAL, "no strip kernel for this shape");
    return cuda_status(wl_launch_fast(L, static_cast<cudaStream_t>(stream)), "fast_kernel");
}

extern "C" {

int wl_dwt2_inverse_strip(const float* ll, const float* hl, const float* lh, const float* hh,
                          int qw, int qrows, int halo_qrows, long plane_pitch, int wavelet,
                          int scheme, int undo_scaling, float* img, long img_pitch,
                          void* stream) {
    return wl_inverse_strip_ex(ll, hl, lh, hh, qw, qrows, halo_qrows, halo_qrows, plane_pitch,
                               wavelet, scheme, undo_scaling, img, img_pitch, stream,
                               WL_PERIODIC);
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

// transform.cpp:198-227: level l transforms the previous level's LL (the
// batched path with one image: same launches).
int wl_dwt2_pyramid_forward(const float* img, int w, int h, int levels, int wavelet, int scheme,
                            int boundary, int scaling, float* pyramid, float* scratch,
                            void* stream) {
    if (levels < 1) return fail(WL_EINVAL, "levels must be >= 1");
    if (w <= 0 || h <= 0) return fail(WL_EINVAL, "forward requires even positive dimensions");
    const int div = 1 << (levels > 30 ? 30 : levels);
    if (levels > 30 || w % div != 0 || h % div != 0)
        return fail(WL_EINVAL, "image dimensions must be divisible by 2^levels");
    if (!img || !pyramid || !scratch) return fail(WL_EINVAL, "null buffer");
    const long n = static_cast<long>(w) * h;
    return wl_dwt2_pyramid_forward_batch(img, w, h, n, 1, levels, wavelet, scheme, boundary,
                                         scaling, pyramid, n, scratch, stream);
}

// transform.cpp:229-256: coarsest level first.
static int pyramid_inverse_impl(const float* pyramid, int w, int h, int levels, int wavelet,
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

size_t wl_pyramid_batch_scratch_elems(int w, int h, int levels, int n) {
    if (w <= 0 || h <= 0 || levels < 1 || n < 1) return 0;
    const size_t q1 = static_cast<size_t>(w / 2) * (h / 2);
    // LL ping-pong: n*q1 (LL of levels 0, 2, ...) | n*q1/4 (levels 1, 3, ...)
    return static_cast<size_t>(n) * (q1 + (levels > 1 ? q1 / 4 : 0));
}

// Batched multi_level_forward (transform.cpp:198-227 per image): one launch
// per level for the whole batch. Image b is at imgs + b*img_stride (pitch w),
// its flat pyramid at pyramids + b*pyr_stride; level LL planes ping-pong in
// `scratch` (wl_pyramid_batch_scratch_elems floats).
static int pyramid_forward_batch_impl(const float* imgs, int w, int h, long img_stride, int n,
                                      int levels, int wavelet, int scheme, int boundary,
                                      int scaling, float* pyramids, long pyr_stride,
                                      float* scratch, void* stream) {
    if (n < 0) return fail(WL_EINVAL, "batch size must be >= 0");
    if (levels < 1) return fail(WL_EINVAL, "levels must be >= 1");
    if (w <= 0 || h <= 0) return fail(WL_EINVAL, "forward requires even positive dimensions");
    if (levels > 30 || w % (1 << levels) != 0 || h % (1 << levels) != 0)
        return fail(WL_EINVAL, "image dimensions must be divisible by 2^levels");
    if (!valid_ids(wavelet, scheme, boundary))
        return fail(WL_EINVAL, "unknown wavelet/scheme/boundary");
    if (n == 0) return WL_OK;
    if (!imgs || !pyramids || !scratch) return fail(WL_EINVAL, "null buffer");
    if (n > 1 && (img_stride < static_cast<long>(w) * h || pyr_stride < static_cast<long>(w) * h))
        return fail(WL_EINVAL, "batch stride too small");
    const size_t q1 = static_cast<size_t>(w / 2) * (h / 2);
    float* ping[2] = {scratch, scratch + static_cast<size_t>(n) * q1};
    size_t offs[32];  // pyramid offset of level l's HL plane
    {
        size_t off = 0;
        for (int l = 0; l < levels; ++l) {
            offs[l] = off;
            off += 3 * static_cast<size_t>(w >> (l + 1)) * (h >> (l + 1));
        }
        offs[levels] = off;  // coarsest LL
    }
    // Level l reading `src` (batch stride src_stride), LL to `ll` (stride ll_stride).
    auto level = [&](int l, const float* src, long src_stride, float* ll, long ll_stride) {
        const int qw = w >> (l + 1), qh = h >> (l + 1);
        const long np = static_cast<long>(qw) * qh;
        float* hl = pyramids + offs[l];
        WlLevel L{};
        L.in[0] = src;
        L.out[0] = ll;
        L.out[1] = hl;
        L.out[2] = hl + np;
        L.out[3] = hl + 2 * np;
        L.qw = qw;
        L.qh = qh;
        L.in_pitch = 2 * qw;
        L.out_pitch = qw;
        L.wavelet = wavelet;
        L.scheme = scheme;
        L.direction = 0;
        L.prog = prog_index(wavelet, scheme, 0);
        L.boundary = boundary;
        L.scaling = scaling != 0;
        L.nb = n;
        L.in_bstride[0] = src_stride;
        L.out_bstride[0] = ll_stride;
        L.out_bstride[1] = L.out_bstride[2] = L.out_bstride[3] = pyr_stride;
        return L;
    };
    // LL of level l: the pyramid's coarsest plane, or scratch buffer `buf` at `at`
    auto ll_of = [&](int l, int buf, size_t at, float** p, long* stride) {
        if (l + 1 == levels) {
            *p = pyramids + offs[levels];
            *stride = pyr_stride;
        } else {
            *p = ping[buf] + at;
            *stride = static_cast<long>(w >> (l + 1)) * (h >> (l + 1));
        }
    };
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const float* src = imgs;
    long src_stride = img_stride;
    int inbuf = -1;  // scratch buffer holding src (-1: the images)
    for (int l = 0; l < levels;) {
        const int q = inbuf == 0 ? 1 : 0;  // the other buffer (LL_l never overwrites its input)
        float* ll;
        long ls;
        ll_of(l, q, 0, &ll, &ls);
        const int st = launch_level_batch(level(l, src, src_stride, ll, ls), s);
        if (st != WL_OK) return st;
        src = ll;
        src_stride = ls;
        inbuf = q;
        ++l;
    }
    return WL_OK;
}

// Batched multi_level_inverse (transform.cpp:229-256 per image).
static int pyramid_inverse_batch_impl(const float* pyramids, int w, int h, long pyr_stride,
                                      int n, int levels, int wavelet, int scheme, int boundary,
                                      int undo_scaling, float* imgs, long img_stride,
                                      float* scratch, void* stream) {
    if (n < 0) return fail(WL_EINVAL, "batch size must be >= 0");
    if (levels < 1) return fail(WL_EINVAL, "levels must be >= 1");
    if (w <= 0 || h <= 0 || levels > 30 || w % (1 << levels) != 0 || h % (1 << levels) != 0)
        return fail(WL_EINVAL, "pyramid level dimensions are inconsistent");
    if (!valid_ids(wavelet, scheme, boundary))
        return fail(WL_EINVAL, "unknown wavelet/scheme/boundary");
    if (n == 0) return WL_OK;
    if (!imgs || !pyramids || !scratch) return fail(WL_EINVAL, "null buffer");
    if (n > 1 && (img_stride < static_cast<long>(w) * h || pyr_stride < static_cast<long>(w) * h))
        return fail(WL_EINVAL, "batch stride too small");
    const size_t q1 = static_cast<size_t>(w / 2) * (h / 2);
    float* ping[2] = {scratch, scratch + static_cast<size_t>(n) * q1};
    long offs[32];
    long off = 0;
    for (int l = 0; l < levels; ++l) {
        offs[l] = off;
        off += 3 * static_cast<long>(w >> (l + 1)) * (h >> (l + 1));
    }
    const float* ll = pyramids + off;  // coarsest LL
    long ll_stride = pyr_stride;
    for (int l = levels - 1; l >= 0; --l) {
        const int qw = w >> (l + 1), qh = h >> (l + 1);
        const long np = static_cast<long>(qw) * qh;
        const float* hl = pyramids + offs[l];
        WlLevel L{};
        L.in[0] = ll;
        L.in[1] = hl;
        L.in[2] = hl + np;
        L.in[3] = hl + 2 * np;
        L.out[0] = l == 0 ? imgs : ping[(l - 1) & 1];
        L.qw = qw;
        L.qh = qh;
        L.in_pitch = qw;
        L.out_pitch = 2 * qw;
        L.wavelet = wavelet;
        L.scheme = scheme;
        L.direction = 1;
        L.prog = prog_index(wavelet, scheme, 1);
        L.boundary = boundary;
        L.scaling = undo_scaling != 0;
        L.nb = n;
        L.in_bstride[0] = ll_stride;
        L.in_bstride[1] = L.in_bstride[2] = L.in_bstride[3] = pyr_stride;
        L.out_bstride[0] = l == 0 ? img_stride : 4 * np;
        const int st = launch_level_batch(L, static_cast<cudaStream_t>(stream));
        if (st != WL_OK) return st;
        ll = L.out[0];
        ll_stride = L.out_bstride[0];
    }
    return WL_OK;
}

}  // extern "C"

// ------------------------------------------------------------ graph cache
// The multi-level drivers (transform.cpp:198-256) issue one launch (plus TMA
// descriptor encodes) per level. A call repeated with identical arguments is
// replayed from a CUDA graph: the first call runs eagerly (and warms every
// lazy per-kernel setup), the second is captured on a thread-local stream
// and instantiated, every later one is one cudaGraphLaunch on the caller's
// stream. Any capture failure falls back to eager launches for that key.
// WL_GRAPHS=0 (or wl_set_graphs(0)) disables it.
namespace {

std::atomic<int> g_graphs{[] {
    const char* v = getenv("WL_GRAPHS");
    return v && v[0] == '0' ? 0 : 1;
}()};

struct GraphKey {
    int fn, device, engine, pad;
    int w, h, n, levels, wavelet, scheme, boundary, scaling;
    const void *a, *b, *c;
    long s1, s2;
    bool operator==(const GraphKey& o) const { return std::memcmp(this, &o, sizeof o) == 0; }
};

struct GraphEntry {
    GraphKey key;
    cudaGraphExec_t exec = nullptr;
    long kernels = 0;  // kernel nodes (added to wl_launch_count per replay)
    int state = 0;     // 0 seen once, 1 captured, 2 eager only
    unsigned long long used = 0;
};

struct GraphCache {
    static constexpr int kMax = 16;
    GraphEntry e[kMax];
    int n = 0;
    unsigned long long tick = 0;
    cudaStream_t cap[64] = {};
    ~GraphCache() {
        for (int i = 0; i < n; ++i)
            if (e[i].exec) cudaGraphExecDestroy(e[i].exec);
    }
    GraphEntry* find(const GraphKey& k) {
        for (int i = 0; i < n; ++i)
            if (e[i].key == k) return &e[i];
        return nullptr;
    }
    GraphEntry* insert(const GraphKey& k) {
        int slot = n < kMax ? n++ : 0;
        if (slot == 0 && n == kMax)
            for (int i = 1; i < kMax; ++i)
                if (e[i].used < e[slot].used) slot = i;
        if (e[slot].exec) cudaGraphExecDestroy(e[slot].exec);
        e[slot] = GraphEntry{};
        e[slot].key = k;
        return &e[slot];
    }
};

thread_local GraphCache g_cache;

template <class F>
int with_graph(GraphKey k, void* stream, F&& run) {
    if (!g_graphs.load()) return run(stream);
    cudaGetDevice(&k.device);
    k.engine = g_engine.load();
    GraphCache& c = g_cache;
    GraphEntry* e = c.find(k);
    if (!e) {
        e = c.insert(k);
        e->used = ++c.tick;
        return run(stream);  // first call: eager
    }
    e->used = ++c.tick;
    if (e->state == 2) return run(stream);
    if (e->state == 0) {
        cudaStream_t& cs = c.cap[k.device & 63];
        if (!cs && cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking) != cudaSuccess) {
            cs = nullptr;
            e->state = 2;
            cudaGetLastError();
            return run(stream);
        }
        const long before = g_launches.load();
        cudaGraph_t g = nullptr;
        int st = WL_ERUNTIME;
        if (cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal) == cudaSuccess) {
            st = run(cs);
            if (cudaStreamEndCapture(cs, &g) != cudaSuccess) st = WL_ERUNTIME;
        }
        g_launches.store(before);  // captured, not launched
        if (st == WL_OK && g && cudaGraphInstantiate(&e->exec, g, 0) == cudaSuccess) {
            size_t nn = 0;
            cudaGraphGetNodes(g, nullptr, &nn);
            std::vector<cudaGraphNode_t> nodes(nn);
            if (nn) cudaGraphGetNodes(g, nodes.data(), &nn);
            for (cudaGraphNode_t nd : nodes) {
                cudaGraphNodeType t;
                if (cudaGraphNodeGetType(nd, &t) == cudaSuccess && t == cudaGraphNodeTypeKernel)
                    ++e->kernels;
            }
            e->state = 1;
        } else {
            e->exec = nullptr;
            e->state = 2;
        }
        if (g) cudaGraphDestroy(g);
        cudaGetLastError();  // clear capture-related errors; eager path reports its own
        if (e->state == 2) return run(stream);
    }
    const cudaError_t le = cudaGraphLaunch(e->exec, static_cast<cudaStream_t>(stream));
    if (le != cudaSuccess) return cuda_status(le, "cudaGraphLaunch");
    g_launches.fetch_add(e->kernels);
    return WL_OK;
}

}  // namespace

extern "C" {

int wl_set_graphs(int on) { return g_graphs.exchange(on ? 1 : 0); }

int wl_dwt2_pyramid_forward_batch(const float* imgs, int w, int h, long img_stride, int n,
                                  int levels, int wavelet, int scheme, int boundary, int scaling,
                                  float* pyramids, long pyr_stride, float* scratch,
                                  void* stream) {
    GraphKey k{};
    k.fn = 1;
    k.w = w; k.h = h; k.n = n; k.levels = levels; k.wavelet = wavelet; k.scheme = scheme;
    k.boundary = boundary; k.scaling = scaling;
    k.a = imgs; k.b = pyramids; k.c = scratch; k.s1 = img_stride; k.s2 = pyr_stride;
    return with_graph(k, stream, [&](void* st) {
        return pyramid_forward_batch_impl(imgs, w, h, img_stride, n, levels, wavelet, scheme,
                                          boundary, scaling, pyramids, pyr_stride, scratch, st);
    });
}

int wl_dwt2_pyramid_inverse_batch(const float* pyramids, int w, int h, long pyr_stride, int n,
                                  int levels, int wavelet, int scheme, int boundary,
                                  int undo_scaling, float* imgs, long img_stride, float* scratch,
                                  void* stream) {
    GraphKey k{};
    k.fn = 2;
    k.w = w; k.h = h; k.n = n; k.levels = levels; k.wavelet = wavelet; k.scheme = scheme;
    k.boundary = boundary; k.scaling = undo_scaling;
    k.a = pyramids; k.b = imgs; k.c = scratch; k.s1 = pyr_stride; k.s2 = img_stride;
    return with_graph(k, stream, [&](void* st) {
        return pyramid_inverse_batch_impl(pyramids, w, h, pyr_stride, n, levels, wavelet, scheme,
                                          boundary, undo_scaling, imgs, img_stride, scratch, st);
    });
}

int wl_dwt2_pyramid_inverse(const float* pyramid, int w, int h, int levels, int wavelet,
                            int scheme, int boundary, int undo_scaling, float* img,
                            float* scratch, void* stream) {
    GraphKey k{};
    k.fn = 3;
    k.w = w; k.h = h; k.n = 1; k.levels = levels; k.wavelet = wavelet; k.scheme = scheme;
    k.boundary = boundary; k.scaling = undo_scaling;
    k.a = pyramid; k.b = img; k.c = scratch;
    return with_graph(k, stream, [&](void* st) {
        return pyramid_inverse_impl(pyramid, w, h, levels, wavelet, scheme, boundary,
                                    undo_scaling, img, scratch, st);
    });
}

}  // extern "C"
