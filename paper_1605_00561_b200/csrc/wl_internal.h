// Internal declarations shared by the kernels and the C-ABI layer.
#pragma once

#include <cuda_runtime.h>

#include "wl_program.h"

// One single-level transform launch (forward: image -> 4 planes; inverse:
// 4 planes -> image). Pitches are in elements.
struct WlLevel {
    const float* in[4];  // fwd: in[0] = image; inv: LL, HL, LH, HH
    float* out[4];       // fwd: LL, HL, LH, HH; inv: out[0] = image
    int qw, qh;          // component-grid (plane) size; image is 2qw x 2qh
    long in_pitch, out_pitch;
    int prog;            // program index ((wavelet*10)+scheme)*2+direction
    int wavelet, scheme, direction;
    int boundary;        // 0 periodic, 1 symmetric
    int scaling;         // apply (fwd) / undo (inv) the zeta^2 scaling step
    // Batch: nb images (0/1 = one), element strides between consecutive
    // images of the input / output buffers (every plane of an image shares
    // its image's offset).
    int nb;
    long in_bstride[4], out_bstride[4];
    // Row window ("strip" mode, fast engine only): only component rows
    // [ylo, yhi) of the qh-row buffer are produced; out[] points at row ylo.
    // yhi == 0: the whole plane (out[] at row 0).
    int ylo, yhi;
    // Strip-pyramid halo wait (wl_strips.cu): when xflag_a is set, the fast
    // engine schedules the window's first and last tile rows last and its
    // producer waits until *xflag_a and *xflag_b reach xepoch (system-scope
    // acquire, timeout -> *xerr) before loading them -- the only tiles that
    // read the halo rows pushed by the neighbour ranks.
    const unsigned* xflag_a;
    const unsigned* xflag_b;
    unsigned xepoch;
    unsigned* xerr;
};

const WlProgram& wl_host_program(int prog);
const WlStep* wl_host_steps();

// Up to 4 rectangles of output cells (the frame around the fast engine's
// tile grid); one CTA per 32x32 tile of each rectangle.
struct WlRects {
    int n;
    int y0[4], x0[4], ny[4], nx[4];
    int ty[4], tx[4];  // tile shape per rectangle (set by wl_launch_interp_rects)
};

// Generic tile interpreter: every wavelet/scheme/direction/boundary.
cudaError_t wl_launch_interp(const WlLevel& L, cudaStream_t stream);
cudaError_t wl_launch_interp_rects(const WlLevel& L, const WlRects& R, cudaStream_t stream);
// Direct 2-D convolution forward (SchemeKind::Convolution): generic
// (every wavelet) and the register/TMA kernel for cdf53/cdf97.
cudaError_t wl_launch_conv(const WlLevel& L, cudaStream_t stream);
cudaError_t wl_launch_conv_fast(const WlLevel& L, cudaStream_t stream);
// Fast register-tile engine; returns cudaErrorNotSupported when the
// (wavelet, scheme, direction) has no fast instantiation.
cudaError_t wl_launch_fast(const WlLevel& L, cudaStream_t stream);
bool wl_fast_supported(const WlLevel& L);
// 0 = no fast instantiation, 1 = TMA path, 2 = direct-load path (no TMA:
// unaligned pitches/pointers, plane widths not = 0 mod 4 cells).
int wl_fast_mode(const WlLevel& L);
// wl_set_engine's value (0 auto, 1 interpreter, 2 fast, 3 fast direct-load).
int wl_engine();

void wl_count_launch();
// Diagnostic per-CTA timestamps (WL_DIAG_TIMES builds; wl_diag_set)
unsigned long long* wl_diag_ptr();
// Records `msg` as this thread's wl_last_error() and returns `code`.
int wl_fail(int code, const char* msg);

// Strip forward with the halo wait folded into the fast engine (wl_strips.cu):
// identical to wl_dwt2_forward_strip, plus WlLevel::xflag_* (null = no wait).
bool wl_strip_wait_capable(int wavelet, int scheme);
int wl_forward_strip_wait(const float* strip, int w, int rows, int halo_rows, long pitch,
                          int wavelet, int scheme, int scaling, float* ll, float* hl, float* lh,
                          float* hh, long plane_pitch, void* stream, const unsigned* xflag_a,
                          const unsigned* xflag_b, unsigned xepoch, unsigned* xerr,
                          int boundary, int halo_top, int halo_bot);

// Can the strip transforms run this shape on dense buffers (pitch = width)
// at 256-byte aligned addresses? forward: w pixels x rows (+ halo_rows above
// and below); inverse (direction 1): w = plane cells, rows = plane rows.
// Asked by the host chunk pipeline and WlStrips BEFORE anything is enqueued.
bool wl_strip_shape_ok(int w, int rows, int halo_rows, int wavelet, int scheme, int direction);
// ... and how: 0 unsupported, 1 fast engine with TMA (halo wait foldable into
// the transform), 2 fast engine direct-load path, 3 convolution kernel.
int wl_strip_mode(int w, int rows, int halo_rows, int wavelet, int scheme, int direction);
// ... for a window with halo_top / halo_bot rows under `boundary` (a
// symmetric window may have 0 halo rows on the image's own edge).
int wl_strip_mode_b(int w, int rows, int halo_top, int halo_bot, int wavelet, int scheme,
                    int direction, int boundary);

// Inverse strip with per-side halo rows and a boundary (a symmetric window
// may have 0 halo rows on the image's own edge); wl_dwt2_inverse_strip is
// the periodic case.
int wl_inverse_strip_ex(const float* ll, const float* hl, const float* lh, const float* hh,
                        int qw, int qrows, int halo_top, int halo_bot, long plane_pitch,
                        int wavelet, int scheme, int undo_scaling, float* img, long img_pitch,
                        void* stream, int boundary);
