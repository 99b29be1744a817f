/*
 * TEST INFRASTRUCTURE -- CPU oracle, NOT the product.
 *
 * Plain-C restatement of the reference hot path (float64):
 * /root/reference/proj/src/transform.cpp. Rows of a step are split over
 * OpenMP threads (like parallel_rows, transform.cpp:36-55); every output
 * element is computed by one thread in the reference's order, so the result
 * is independent of the thread count (OMP_NUM_THREADS). Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline leg may load this library, and only as the
 * checker. It is pinned against the unmodified reference (oracle/_ref) and
 * against the golden fixtures in tests/golden/ (see tests/test_oracle.py).
 *
 * A step matrix is passed as a flat tap list in the reference's summation
 * order (transform.cpp:103-116: destination component, then source component
 * 0..3, then std::map order of the (k_m, k_n) exponent pair). Each tap is
 * five ints {dst, src, k_m, k_n, is_identity} plus a double coefficient; an
 * is_identity tap is the "diagonal entry equal to one" shortcut of
 * transform.cpp:106-109 (acc += x without a multiply).
 */
#include <stddef.h>
#include <stdlib.h>
#include <string.h>

enum { LL = 0, HL = 1, LH = 2, HH = 3 };

/* transform.cpp:59-72 resolve_index: periodic wrap or whole-point mirror
 * (iterated), n == 1 absorbs every index. */
/* Worker threads of the parallel row loops (1 without OpenMP). */
#ifdef _OPENMP
#include <omp.h>
int wlo_threads(void) { return omp_get_max_threads(); }
#else
int wlo_threads(void) { return 1; }
#endif

int wlo_resolve_index(int i, int n, int boundary) {
    if (i >= 0 && i < n) return i;
    if (n == 1) return 0;
    if (boundary == 0) {
        int m = i % n;
        return m < 0 ? m + n : m;
    }
    while (i < 0 || i >= n) {
        if (i < 0) i = -i;
        if (i >= n) i = 2 * (n - 1) - i;
    }
    return i;
}

/* transform.cpp:74-86 polyphase_split: LL<-(2r,2c) HL<-(2r,2c+1)
 * LH<-(2r+1,2c) HH<-(2r+1,2c+1). q4 holds the 4 planes back to back. */
void wlo_split(const double* img, int w, int h, double* q4) {
    const int qw = w / 2, qh = h / 2;
    const size_t n = (size_t)qw * qh;
    for (int r = 0; r < qh; ++r)
        for (int c = 0; c < qw; ++c) {
            const size_t o = (size_t)r * qw + c;
            q4[LL * n + o] = img[(size_t)(2 * r) * w + 2 * c];
            q4[HL * n + o] = img[(size_t)(2 * r) * w + 2 * c + 1];
            q4[LH * n + o] = img[(size_t)(2 * r + 1) * w + 2 * c];
            q4[HH * n + o] = img[(size_t)(2 * r + 1) * w + 2 * c + 1];
        }
}

/* transform.cpp:88-98 polyphase_merge (exact inverse of the split). */
void wlo_merge(const double* q4, int qw, int qh, double* img) {
    const int w = 2 * qw;
    const size_t n = (size_t)qw * qh;
    for (int r = 0; r < qh; ++r)
        for (int c = 0; c < qw; ++c) {
            const size_t o = (size_t)r * qw + c;
            img[(size_t)(2 * r) * w + 2 * c] = q4[LL * n + o];
            img[(size_t)(2 * r) * w + 2 * c + 1] = q4[HL * n + o];
            img[(size_t)(2 * r + 1) * w + 2 * c] = q4[LH * n + o];
            img[(size_t)(2 * r + 1) * w + 2 * c + 1] = q4[HH * n + o];
        }
}

/* transform.cpp:100-125 apply_step: out-of-place y_i = sum_j M_ij (*) x_j,
 * a term z_m^km z_n^kn reading x_j[r - kn][c - km] under the boundary. */
void wlo_apply_step(const double* in4, int qw, int qh, const int* taps, const double* coeff,
                    int ntaps, int boundary, double* out4) {
    const size_t n = (size_t)qw * qh;
    for (int comp = 0; comp < 4; ++comp) {
        int t0 = 0, t1;
        while (t0 < ntaps && taps[5 * t0] != comp) ++t0;
        t1 = t0;
        while (t1 < ntaps && taps[5 * t1] == comp) ++t1;
#pragma omp parallel for schedule(static)
        for (int r = 0; r < qh; ++r)
            for (int c = 0; c < qw; ++c) {
                double acc = 0.0;
                for (int t = t0; t < t1; ++t) {
                    const int* tp = taps + 5 * t;
                    const double* x = in4 + (size_t)tp[1] * n;
                    if (tp[4]) {
                        acc += x[(size_t)r * qw + c];
                        continue;
                    }
                    const int rr = wlo_resolve_index(r - tp[3], qh, boundary);
                    const int cc = wlo_resolve_index(c - tp[2], qw, boundary);
                    acc += coeff[t] * x[(size_t)rr * qw + cc];
                }
                out4[(size_t)comp * n + (size_t)r * qw + c] = acc;
            }
    }
}

/* transform.cpp:154-159 scale_planes: LL *= s, HH /= s, s = zeta^2 (or its
 * reciprocal when inverting). */
void wlo_scale(double* q4, size_t n, double zeta, int invert) {
    if (zeta == 1.0) return;
    const double s = invert ? 1.0 / (zeta * zeta) : zeta * zeta;
    for (size_t i = 0; i < n; ++i) q4[LL * n + i] *= s;
    for (size_t i = 0; i < n; ++i) q4[HH * n + i] /= s;
}

/* Runs a step list (step_ntaps[k] taps each, concatenated). */
static void run_steps(double* cur, double* tmp, int qw, int qh, int nsteps, const int* step_ntaps,
                      const int* taps, const double* coeff, int boundary, double** result) {
    const size_t n4 = (size_t)4 * qw * qh;
    double* a = cur;
    double* b = tmp;
    int off = 0;
    for (int k = 0; k < nsteps; ++k) {
        wlo_apply_step(a, qw, qh, taps + 5 * off, coeff + off, step_ntaps[k], boundary, b);
        off += step_ntaps[k];
        double* t = a;
        a = b;
        b = t;
    }
    (void)n4;
    *result = a;
}

/* transform.cpp:163-176 forward (lifting kinds): split, every step in order,
 * optional scaling. Returns 1 on invalid dimensions (invalid_argument). */
int wlo_forward_steps(const double* img, int w, int h, int nsteps, const int* step_ntaps,
                      const int* taps, const double* coeff, int boundary, int scaling, double zeta,
                      double* out4) {
    if (w <= 0 || h <= 0 || w % 2 || h % 2) return 1;
    const int qw = w / 2, qh = h / 2;
    const size_t n = (size_t)qw * qh;
    double* a = (double*)malloc(4 * n * sizeof(double));
    double* b = (double*)malloc(4 * n * sizeof(double));
    double* res;
    wlo_split(img, w, h, a);
    run_steps(a, b, qw, qh, nsteps, step_ntaps, taps, coeff, boundary, &res);
    if (scaling) wlo_scale(res, n, zeta, 0);
    memcpy(out4, res, 4 * n * sizeof(double));
    free(a);
    free(b);
    return 0;
}

/* transform.cpp:129-152 forward_convolution: the four 2-D analysis filters
 * evaluated at subsampled positions, mirrored on the IMAGE grid. Filter k
 * has ntap[k] taps {km, kn} (ints, 2 per tap) with coefficients. */
int wlo_forward_conv(const double* img, int w, int h, const int* ntap, const int* taps,
                     const double* coeff, int boundary, int scaling, double zeta, double* out4) {
    if (w <= 0 || h <= 0 || w % 2 || h % 2) return 1;
    const int qw = w / 2, qh = h / 2;
    const size_t n = (size_t)qw * qh;
    static const int row_phase[4] = {0, 0, 1, 1};
    static const int col_phase[4] = {0, 1, 0, 1};
    int off = 0;
    for (int comp = 0; comp < 4; ++comp) {
#pragma omp parallel for schedule(static)
        for (int r = 0; r < qh; ++r)
            for (int c = 0; c < qw; ++c) {
                double acc = 0.0;
                for (int t = off; t < off + ntap[comp]; ++t) {
                    const int rr = wlo_resolve_index(2 * r + row_phase[comp] - taps[2 * t + 1], h,
                                                     boundary);
                    const int cc = wlo_resolve_index(2 * c + col_phase[comp] - taps[2 * t], w,
                                                     boundary);
                    acc += coeff[t] * img[(size_t)rr * w + cc];
                }
                out4[comp * n + (size_t)r * qw + c] = acc;
            }
        off += ntap[comp];
    }
    if (scaling) wlo_scale(out4, n, zeta, 0);
    return 0;
}

/* transform.cpp:178-196 inverse: undo scaling, run the given inverse step
 * list (the reference's is the reversed negated Sweldens list), merge. */
int wlo_inverse_steps(const double* in4, int qw, int qh, int nsteps, const int* step_ntaps,
                      const int* taps, const double* coeff, int boundary, int undo, double zeta,
                      double* img) {
    if (qw <= 0 || qh <= 0) return 1;
    const size_t n = (size_t)qw * qh;
    double* a = (double*)malloc(4 * n * sizeof(double));
    double* b = (double*)malloc(4 * n * sizeof(double));
    double* res;
    memcpy(a, in4, 4 * n * sizeof(double));
    if (undo) wlo_scale(a, n, zeta, 1);
    run_steps(a, b, qw, qh, nsteps, step_ntaps, taps, coeff, boundary, &res);
    wlo_merge(res, qw, qh, img);
    free(a);
    free(b);
    return 0;
}

/* transform.cpp:198-227 multi_level_forward, lifting kinds. Flat output:
 * per level (finest first) HL, LH, HH, then the coarsest LL. */
int wlo_pyramid_forward_steps(const double* img, int w, int h, int levels, int nsteps,
                              const int* step_ntaps, const int* taps, const double* coeff,
                              int boundary, int scaling, double zeta, double* out) {
    if (levels < 1) return 1;
    if (w % (1 << levels) || h % (1 << levels) || w <= 0 || h <= 0) return 1;
    double* cur = (double*)malloc((size_t)w * h * sizeof(double));
    double* q = (double*)malloc((size_t)w * h * sizeof(double));
    memcpy(cur, img, (size_t)w * h * sizeof(double));
    double* o = out;
    int cw = w, ch = h;
    for (int l = 0; l < levels; ++l) {
        const size_t n = (size_t)(cw / 2) * (ch / 2);
        wlo_forward_steps(cur, cw, ch, nsteps, step_ntaps, taps, coeff, boundary, scaling, zeta, q);
        memcpy(o, q + n, 3 * n * sizeof(double));
        o += 3 * n;
        memcpy(cur, q, n * sizeof(double));
        cw /= 2;
        ch /= 2;
    }
    memcpy(o, cur, (size_t)cw * ch * sizeof(double));
    free(cur);
    free(q);
    return 0;
}

/* transform.cpp:229-256 multi_level_inverse on the flat layout above. */
int wlo_pyramid_inverse_steps(const double* in, int w, int h, int levels, int nsteps,
                              const int* step_ntaps, const int* taps, const double* coeff,
                              int boundary, int undo, double zeta, double* img) {
    if (levels < 1) return 1;
    size_t offs[32];
    size_t off = 0;
    int pw = w / 2, ph = h / 2;
    for (int l = 0; l < levels; ++l) {
        offs[l] = off;
        off += 3 * (size_t)pw * ph;
        if (l + 1 < levels) {
            pw /= 2;
            ph /= 2;
        }
    }
    double* ll = (double*)malloc((size_t)w * h * sizeof(double));
    double* q = (double*)malloc((size_t)w * h * sizeof(double));
    memcpy(ll, in + off, (size_t)pw * ph * sizeof(double));
    for (int l = levels - 1; l >= 0; --l) {
        const size_t n = (size_t)pw * ph;
        memcpy(q, ll, n * sizeof(double));
        memcpy(q + n, in + offs[l], 3 * n * sizeof(double));
        wlo_inverse_steps(q, pw, ph, nsteps, step_ntaps, taps, coeff, boundary, undo, zeta, ll);
        pw *= 2;
        ph *= 2;
    }
    memcpy(img, ll, (size_t)w * h * sizeof(double));
    free(ll);
    free(q);
    return 0;
}
