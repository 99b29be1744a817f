/*
 * wl_dwt.h -- C-ABI of the B200-native 2-D lifting DWT (libwavelift_b200.so).
 *
 * Drop-in boundary for the reference's transform API
 * (/root/reference/proj/include/wavelift/transform.hpp). Every entry point
 * takes plain pointers and sizes; image and subband buffers are caller-owned
 * DEVICE memory (float32, row-major, pitches in ELEMENTS) and work is
 * enqueued on the caller's CUDA stream (NULL = legacy default stream).
 * Host-buffer (float64 Image/QuadGrid/Pyramid) parity wrappers live in the
 * C++ header wavelift_b200.hpp on top of this ABI.
 *
 * Enumerations follow the reference:
 *   wavelet  : WL_CDF53, WL_CDF97, WL_DD137            (wavelets.cpp:27-62)
 *   scheme   : SchemeKind order                        (schemes.hpp:15-26)
 *   boundary : WL_PERIODIC, WL_SYMMETRIC               (transform.hpp:44)
 * Status codes mirror the reference's exception classes
 * (wavelift_main.cpp:363-369): WL_OK, WL_EINVAL (std::invalid_argument),
 * WL_ERUNTIME (CUDA / other runtime failure). wl_last_error() returns the
 * message of the calling thread's last failure.
 */
#ifndef WL_DWT_H_
#define WL_DWT_H_

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { WL_OK = 0, WL_EINVAL = 1, WL_ERUNTIME = 2 };
enum { WL_CDF53 = 0, WL_CDF97 = 1, WL_DD137 = 2 };
enum {
    WL_SWELDENS = 0, WL_IWAHASHI, WL_IWAHASHI_STAR, WL_EXPLOSIVE, WL_EXPLOSIVE_STAR,
    WL_MONOLITHIC, WL_MONOLITHIC_STAR, WL_POLYPHASE, WL_POLYPHASE_STAR, WL_CONVOLUTION
};
enum { WL_PERIODIC = 0, WL_SYMMETRIC = 1 };
enum { WL_FORWARD = 0, WL_INVERSE = 1 };

/* Message of this thread's last non-OK status (empty string if none). */
const char* wl_last_error(void);
/* Library version / build string. */
const char* wl_version(void);

/* Cost and structure of a (wavelet, scheme, direction) program:
 * barriers = count_barriers (schemes.cpp:193-198), macs = count_macs
 * (schemes.cpp:176-191), epochs = block barriers per tile in the kernel,
 * halo = tile halo in component cells (parsim.cpp:185-218 required_halo).
 * Replaces schemes.hpp:58-62. */
int wl_scheme_info(int wavelet, int scheme, int direction, int* barriers, long* macs,
                   int* epochs, int* halo);

/* ------------------------------------------------- scheme structure (host)
 * The result of build_scheme(kind, wavelet) (schemes.cpp:146-174,
 * schemes.hpp:34-45) for callers that walk Scheme::steps (e.g. parsim.cpp:
 * 250,285-286,337-338). matrix_kind follows MatrixKind (polyphase.hpp:24-38:
 * T_H=0 ... N_FULL=12). A term is one Laurent monomial of entry (row, col):
 * coefficient * z_m^km * z_n^kn; terms come in the reference's order (row,
 * col, then std::map order of (km, kn)). */
/* Number of steps (0 for Convolution), -1 for unknown ids. */
int wl_scheme_nsteps(int wavelet, int scheme);
/* Step k: MatrixKind, needs_barrier, number of terms, label (NUL-terminated,
 * truncated to label_cap). Any output pointer may be NULL. */
int wl_scheme_step(int wavelet, int scheme, int k, int* matrix_kind, int* needs_barrier,
                   int* nterms, char* label, int label_cap);
/* Terms of step k into arrays of `cap` entries (any may be NULL). Returns the
 * number of terms (call with cap = 0 to size the arrays), -1 on bad ids. */
int wl_scheme_step_terms(int wavelet, int scheme, int k, int* rows, int* cols, int* km, int* kn,
                         double* coeff, int cap);
/* Convolution: 2-D analysis filter `which` (0 f_ll, 1 f_hl, 2 f_lh, 3 f_hh;
 * wavelets.cpp:80-88, wavelets.hpp:50-53) as km/kn/coeff terms in map order.
 * Returns the number of taps (cap = 0 to size), -1 on bad ids. */
int wl_scheme_conv_filter(int wavelet, int which, int* km, int* kn, double* coeff, int cap);

/* One step matrix on device planes, out of place: replaces `QuadGrid
 * apply_step(const QuadGrid&, const StepMatrix&, BoundaryMode)`
 * (transform.hpp:57-60, transform.cpp:100-125). The matrix is given as
 * `nterms` HOST terms (rows/cols/km/kn/coeff as above, <= 512); a term reads
 * the source plane at (r - kn, c - km) resolved under `boundary`. Sums per
 * destination in (source, map) order with unfused multiply/add, float32. */
int wl_apply_step(const float* ll, const float* hl, const float* lh, const float* hh, int qw,
                  int qh, long pitch, int nterms, const int* rows, const int* cols, const int* km,
                  const int* kn, const double* coeff, int boundary, float* out_ll, float* out_hl,
                  float* out_lh, float* out_hh, long out_pitch, void* stream);

/* transform.cpp:59-72 resolve_index (host-side helper). */
int wl_resolve_index(int i, int n, int boundary);

/* One level, forward: replaces `QuadGrid forward(const Image&, const Scheme&,
 * BoundaryMode, bool apply_scaling)` (transform.hpp:65-66, transform.cpp:163-176).
 * img: w x h (even, positive), img_pitch >= w. Output planes LL, HL, LH, HH are
 * (w/2) x (h/2) with plane_pitch >= w/2. */
int wl_dwt2_forward(const float* img, int w, int h, long img_pitch, int wavelet, int scheme,
                    int boundary, int scaling, float* ll, float* hl, float* lh, float* hh,
                    long plane_pitch, void* stream);

/* One level, inverse: replaces `Image inverse(const QuadGrid&, const
 * WaveletSpec&, BoundaryMode, bool undo_scaling)` (transform.hpp:71-72,
 * transform.cpp:178-196). `scheme` selects the inverse kernel: WL_SWELDENS is
 * the reference's own algorithm (reversed negated separable steps); every
 * other lifting scheme runs its own reversed, inverted step list with the
 * same barrier count as its forward (identical result under the periodic
 * boundary; see DESIGN.md for the symmetric-boundary semantics).
 * WL_CONVOLUTION maps to WL_SWELDENS. */
int wl_dwt2_inverse(const float* ll, const float* hl, const float* lh, const float* hh, int qw,
                    int qh, long plane_pitch, int wavelet, int scheme, int boundary,
                    int undo_scaling, float* img, long img_pitch, void* stream);

/* Multi-level pyramid, replaces multi_level_forward / multi_level_inverse
 * (transform.hpp:87-91, transform.cpp:198-256). Flat pyramid layout (device,
 * densely packed): for each level l = 0..levels-1 (finest first) the HL, LH, HH
 * planes of (w>>(l+1)) x (h>>(l+1)), then the coarsest LL plane -- the
 * subband_io payload order (subband_io.hpp:7-20). `scratch` must hold
 * wl_pyramid_scratch_elems(w, h, levels) floats. */
size_t wl_pyramid_elems(int w, int h, int levels);
size_t wl_pyramid_scratch_elems(int w, int h, int levels);
int wl_dwt2_pyramid_forward(const float* img, int w, int h, int levels, int wavelet, int scheme,
                            int boundary, int scaling, float* pyramid, float* scratch,
                            void* stream);
int wl_dwt2_pyramid_inverse(const float* pyramid, int w, int h, int levels, int wavelet,
                            int scheme, int boundary, int undo_scaling, float* img,
                            float* scratch, void* stream);

/* ---------------------------------------------------------------- batches
 * BASELINE configs[4] (independent images). The reference transforms one
 * Image per call (transform.cpp:163, :198); these run the same per-image
 * transform over n images in ONE launch per level (3-D TMA boxes). Image b
 * lives at img + b*img_stride; its planes at ll/hl/lh/hh + b*plane_stride.
 * Results are identical to n single-image calls. */
int wl_dwt2_forward_batch(const float* img, int w, int h, long img_pitch, long img_stride,
                          int n, int wavelet, int scheme, int boundary, int scaling, float* ll,
                          float* hl, float* lh, float* hh, long plane_pitch, long plane_stride,
                          void* stream);
int wl_dwt2_inverse_batch(const float* ll, const float* hl, const float* lh, const float* hh,
                          int qw, int qh, long plane_pitch, long plane_stride, int n, int wavelet,
                          int scheme, int boundary, int undo_scaling, float* img, long img_pitch,
                          long img_stride, void* stream);
/* Batched multi_level_forward / multi_level_inverse (transform.cpp:198-256
 * per image): images dense (pitch w) at img_stride apart, flat pyramids
 * (wl_dwt2_pyramid_forward layout) at pyr_stride apart; `scratch` holds
 * wl_pyramid_batch_scratch_elems(w, h, levels, n) floats. */
size_t wl_pyramid_batch_scratch_elems(int w, int h, int levels, int n);
int wl_dwt2_pyramid_forward_batch(const float* imgs, int w, int h, long img_stride, int n,
                                  int levels, int wavelet, int scheme, int boundary, int scaling,
                                  float* pyramids, long pyr_stride, float* scratch, void* stream);
int wl_dwt2_pyramid_inverse_batch(const float* pyramids, int w, int h, long pyr_stride, int n,
                                  int levels, int wavelet, int scheme, int boundary,
                                  int undo_scaling, float* imgs, long img_stride, float* scratch,
                                  void* stream);

/* ------------------------------------------------------------- row strips
 * BASELINE configs[3]: one image split into row strips (one per GPU). A strip
 * transform computes the rows of `forward` / `inverse` (periodic boundary)
 * that belong to the strip, bit-identical to the whole-image call, given
 * `halo` rows of the neighbouring strips physically present above and below
 * the strip in its buffer. cdf53/cdf97 only (the fast engine / convolution
 * kernel); 16-byte aligned buffers and pitches.
 * wl_strip_halo_rows: minimum halo -- pixel rows (direction 0) or plane rows
 * (direction 1); -1 for an unsupported wavelet. */
int wl_strip_halo_rows(int wavelet, int scheme, int direction);
/* strip: first interior row; rows [-halo_rows, rows + halo_rows) readable.
 * Output planes: rows/2 rows of (w/2). */
int wl_dwt2_forward_strip(const float* strip, int w, int rows, int halo_rows, long pitch,
                          int wavelet, int scheme, int scaling, float* ll, float* hl, float* lh,
                          float* hh, long plane_pitch, void* stream);
/* planes: first interior plane row; rows [-halo_qrows, qrows + halo_qrows)
 * readable. Output: 2*qrows image rows of 2*qw pixels. */
int wl_dwt2_inverse_strip(const float* ll, const float* hl, const float* lh, const float* hh,
                          int qw, int qrows, int halo_qrows, long plane_pitch, int wavelet,
                          int scheme, int undo_scaling, float* img, long img_pitch,
                          void* stream);

/* Row-strip multi-level pyramid across ranks (one process per GPU):
 * replaces multi_level_forward (transform.cpp:198-227) for one image whose
 * rows are split evenly over `nranks` ranks (rank r owns image rows
 * [r*h/nranks, (r+1)*h/nranks)), periodic boundary. Every level exchanges
 * `wl_strip_halo_rows` rows with the two neighbour strips by peer-memory
 * stores into their buffers (CUDA IPC over NVLink) and device-side flags; no
 * host synchronisation or collective library in the level loop.
 *   create -> export (IPC blob, wl_strips_blob_bytes() bytes) -> exchange
 *   blobs out of band -> connect(up = rank-1, down = rank+1, ring) -> fill
 *   wl_strips_input (rows x w, pitch w) -> forward (stream-ordered; every
 *   rank calls it the same number of times) -> check after a sync.
 * The rank's pyramid slice: for each level l, its rows of HL, LH, HH
 * ((rows>>(l+1)) x (w>>(l+1)) each), then its rows of the coarsest LL;
 * wl_strips_slice_elems() floats. Stitching the ranks' slices plane by plane
 * gives exactly wl_dwt2_pyramid_forward's output. */
typedef struct WlStrips WlStrips;
const char* wl_strips_last_error(void);
size_t wl_strips_blob_bytes(void);
int wl_strips_create(int w, int h, int rank, int nranks, int levels, int wavelet, int scheme,
                     int scaling, WlStrips** out);
/* ... with a boundary: WL_SYMMETRIC strips are not a ring -- rank 0 and rank
 * nranks-1 sit on the image's top / bottom edge (per-step mirroring there,
 * transform.cpp:59-72); lifting schemes only. wl_strips_create is
 * WL_PERIODIC. */
int wl_strips_create_ex(int w, int h, int rank, int nranks, int levels, int wavelet, int scheme,
                        int boundary, int scaling, WlStrips** out);
int wl_strips_export(WlStrips* s, void* blob);
int wl_strips_connect(WlStrips* s, const void* up_blob, const void* down_blob);
float* wl_strips_input(WlStrips* s);
size_t wl_strips_slice_elems(const WlStrips* s);
int wl_strips_forward(WlStrips* s, float* slice, void* stream);
/* multi_level_inverse (transform.cpp:229-256) of the rank's slice (the
 * layout wl_strips_forward writes; `undo_scaling` = the create's scaling):
 * writes the rank's rows x w rows of the reconstructed image (pitch w).
 * Coarsest level first; per level `wl_strip_halo_rows(.., 1)` plane rows of
 * all 4 planes are pushed to each neighbour over peer memory. Every rank
 * calls it the same number of times, in the same order as forward. The
 * scheme selects the inverse kernel (Convolution: the Sweldens inverse). */
int wl_strips_inverse(WlStrips* s, const float* slice, float* out_rows, void* stream);
/* WL_ERUNTIME if a halo wait timed out (call after synchronising). */
int wl_strips_check(WlStrips* s);
int wl_strips_destroy(WlStrips* s);

/* ------------------------------------------------------------ host buffers
 * The reference's own call shape: `forward(const Image&)` / `inverse(const
 * QuadGrid&)` take and return HOST memory (transform.hpp:65-72). These take
 * float32 host buffers (pitches in elements), run on the current device and
 * return when the result is in host memory. Periodic cdf53/cdf97 transforms
 * are pipelined in row chunks (strip transforms on 3 streams: H2D, kernels
 * and D2H overlap); everything else runs whole-image. Pin the host buffers
 * (cudaHostAlloc / cudaHostRegister) for asynchronous copies. */
int wl_dwt2_forward_host(const float* img, int w, int h, long img_pitch, int wavelet, int scheme,
                         int boundary, int scaling, float* ll, float* hl, float* lh, float* hh,
                         long plane_pitch);
int wl_dwt2_inverse_host(const float* ll, const float* hl, const float* lh, const float* hh,
                         int qw, int qh, long plane_pitch, int wavelet, int scheme, int boundary,
                         int undo_scaling, float* img, long img_pitch);

/* Engine selection for tests/benchmarks: 0 = auto (fast register-tile engine
 * where available, generic tile interpreter otherwise), 1 = force the generic
 * interpreter, 2 = force the fast engine (WL_EINVAL where unsupported).
 * Returns the previous value. Process-global. */
int wl_set_engine(int engine);
/* Pyramid drivers (wl_dwt2_pyramid_*): a call repeated with identical
 * arguments is replayed from a CUDA graph captured on its second occurrence
 * (one cudaGraphLaunch instead of one launch per level). 1 = on (default;
 * environment WL_GRAPHS=0 turns it off). Returns the previous value. */
int wl_set_graphs(int on);
/* Number of kernel launches this library issued so far (process-global;
 * a graph replay counts its kernel nodes). */
long wl_launch_count(void);
/* Tuning diagnostics only (no reference counterpart): a device buffer of
 * 4 x grid uint64 that a -DWL_DIAG_TIMES build of the fast engine fills per
 * CTA (entry, first tile ready, exit in %globaltimer ns, tiles processed).
 * NULL (default) disables; production builds ignore it. */
void wl_diag_set(void* dev_buf);

#ifdef __cplusplus
}
#endif

#endif /* WL_DWT_H_ */
