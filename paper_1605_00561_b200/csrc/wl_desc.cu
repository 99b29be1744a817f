// Scheme structure queries and apply_step (include/wl_dwt.h):
//
// * wl_scheme_nsteps / wl_scheme_step / wl_scheme_step_terms /
//   wl_scheme_conv_filter expose build_scheme()'s result (schemes.cpp:146-174,
//   schemes.hpp:34-45): the steps with their labels, MatrixKind and
//   needs_barrier flags, every matrix entry's Laurent terms (double), and the
//   four 2-D filters of the Convolution scheme (wavelets.cpp:80-88). Host-only
//   lookups of the tables tools/gen_steps.py generates from schemes.py (which
//   is checked entry by entry against the reference's own dump).
// * wl_apply_step runs ONE step matrix on device planes, out of place, with
//   the reference's per-read boundary resolution and summation order
//   (transform.cpp:100-125): the generic building block a caller that walks
//   Scheme::steps needs (the transforms themselves never call it -- their
//   kernels fuse every step of a scheme).
#include <cstring>

#include "../../include/wl_dwt.h"
#include "gen/scheme_desc_gen.h"
#include "wl_internal.h"

namespace {

constexpr int kNumWavelets = 3, kNumSchemes = 10;

const WlDescScheme* desc(int wavelet, int scheme) {
    if (wavelet < 0 || wavelet >= kNumWavelets || scheme < 0 || scheme >= kNumSchemes)
        return nullptr;
    return &kDescSchemes[wavelet * kNumSchemes + scheme];
}

constexpr int kMaxTerms = 512;

struct ApplyTerm {
    signed char dst, src;
    signed char one;  // diagonal entry equal to 1: acc += x (transform.cpp:109-111)
    signed char pad;
    short dr, dc;     // read offset (row - k_n, col - k_m)
    float c;
};

struct ApplyArgs {
    const float* in[4];
    float* out[4];
    long in_pitch, out_pitch;
    int qw, qh, boundary, nterms;
    int t0[5];  // terms of destination d: [t0[d], t0[d + 1])
    ApplyTerm t[kMaxTerms];
};

__device__ __forceinline__ int resolve(int i, int n, int boundary) {
    if (i >= 0 && i < n) return i;
    if (n == 1) return 0;
    if (boundary == 0) {
        const int m = i % n;
        return m < 0 ? m + n : m;
    }
    while (i < 0 || i >= n) {
        if (i < 0) i = -i;
        if (i >= n) i = 2 * (n - 1) - i;
    }
    return i;
}

// One thread per (cell, destination component); unfused multiply and add
// like the reference's `acc += coeff * x` (no contraction).
__global__ void apply_step_kernel(const __grid_constant__ ApplyArgs a) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    const int r = blockIdx.y;
    const int d = blockIdx.z;
    if (c >= a.qw) return;
    float acc = 0.f;
    for (int k = a.t0[d]; k < a.t0[d + 1]; ++k) {
        const ApplyTerm& t = a.t[k];
        if (t.one) {
            acc = __fadd_rn(acc, a.in[t.src][(long)r * a.in_pitch + c]);
            continue;
        }
        const int rr = resolve(r + t.dr, a.qh, a.boundary);
        const int cc = resolve(c + t.dc, a.qw, a.boundary);
        acc = __fadd_rn(acc, __fmul_rn(t.c, a.in[t.src][(long)rr * a.in_pitch + cc]));
    }
    a.out[d][(long)r * a.out_pitch + c] = acc;
}

}  // namespace

extern "C" {

int wl_scheme_nsteps(int wavelet, int scheme) {
    const WlDescScheme* s = desc(wavelet, scheme);
    if (!s) return wl_fail(WL_EINVAL, "unknown wavelet/scheme"), -1;
    return s->nsteps;
}

int wl_scheme_step(int wavelet, int scheme, int k, int* matrix_kind, int* needs_barrier,
                   int* nterms, char* label, int label_cap) {
    const WlDescScheme* s = desc(wavelet, scheme);
    if (!s) return wl_fail(WL_EINVAL, "unknown wavelet/scheme");
    if (k < 0 || k >= s->nsteps) return wl_fail(WL_EINVAL, "step index out of range");
    const WlDescStep& st = kDescSteps[s->step0 + k];
    if (matrix_kind) *matrix_kind = st.kind;
    if (needs_barrier) *needs_barrier = st.barrier;
    if (nterms) *nterms = st.nterms;
    if (label && label_cap > 0) {
        strncpy(label, st.label, static_cast<size_t>(label_cap) - 1);
        label[label_cap - 1] = '\0';
    }
    return WL_OK;
}

int wl_scheme_step_terms(int wavelet, int scheme, int k, int* rows, int* cols, int* km, int* kn,
                         double* coeff, int cap) {
    const WlDescScheme* s = desc(wavelet, scheme);
    if (!s) return wl_fail(WL_EINVAL, "unknown wavelet/scheme"), -1;
    if (k < 0 || k >= s->nsteps) return wl_fail(WL_EINVAL, "step index out of range"), -1;
    const WlDescStep& st = kDescSteps[s->step0 + k];
    if (cap < st.nterms) return st.nterms;  // ask again with room for every term
    for (int i = 0; i < st.nterms; ++i) {
        const WlDescTerm& t = kDescTerms[st.term0 + i];
        if (rows) rows[i] = t.row;
        if (cols) cols[i] = t.col;
        if (km) km[i] = t.km;
        if (kn) kn[i] = t.kn;
        if (coeff) coeff[i] = t.c;
    }
    return st.nterms;
}

int wl_scheme_conv_filter(int wavelet, int which, int* km, int* kn, double* coeff, int cap) {
    const WlDescScheme* s = desc(wavelet, WL_CONVOLUTION);
    if (!s || which < 0 || which > 3 || s->filter0 < 0)
        return wl_fail(WL_EINVAL, "unknown wavelet/filter"), -1;
    const WlDescFilter& f = kDescFilters[s->filter0 + which];
    if (cap < f.nterms) return f.nterms;
    for (int i = 0; i < f.nterms; ++i) {
        const WlDescTerm& t = kDescTerms[f.term0 + i];
        if (km) km[i] = t.km;
        if (kn) kn[i] = t.kn;
        if (coeff) coeff[i] = t.c;
    }
    return f.nterms;
}

int wl_apply_step(const float* ll, const float* hl, const float* lh, const float* hh, int qw,
                  int qh, long pitch, int nterms, const int* rows, const int* cols, const int* km,
                  const int* kn, const double* coeff, int boundary, float* out_ll, float* out_hl,
                  float* out_lh, float* out_hh, long out_pitch, void* stream) {
    if (qw <= 0 || qh <= 0) return wl_fail(WL_EINVAL, "apply_step requires positive plane dimensions");
    if (boundary < 0 || boundary > 1) return wl_fail(WL_EINVAL, "unknown boundary");
    if (nterms < 0 || nterms > kMaxTerms) return wl_fail(WL_EINVAL, "too many step terms (max 512)");
    if (nterms > 0 && (!rows || !cols || !km || !kn || !coeff))
        return wl_fail(WL_EINVAL, "null term array");
    if (!ll || !hl || !lh || !hh || !out_ll || !out_hl || !out_lh || !out_hh)
        return wl_fail(WL_EINVAL, "null buffer");
    if (pitch < qw || out_pitch < qw) return wl_fail(WL_EINVAL, "pitch too small");
    // ~6 KB parameter block (kernel parameters may be up to 32 KB): built here,
    // copied by the launch
    static thread_local ApplyArgs A;
    A.in[0] = ll; A.in[1] = hl; A.in[2] = lh; A.in[3] = hh;
    A.out[0] = out_ll; A.out[1] = out_hl; A.out[2] = out_lh; A.out[3] = out_hh;
    A.in_pitch = pitch;
    A.out_pitch = out_pitch;
    A.qw = qw;
    A.qh = qh;
    A.boundary = boundary;
    // Terms grouped by destination row, then source column, keeping the
    // caller's order inside an entry (the reference's std::map order).
    int n = 0;
    for (int d = 0; d < 4; ++d) {
        A.t0[d] = n;
        for (int src = 0; src < 4; ++src) {
            int cnt = 0, first = -1;
            for (int i = 0; i < nterms; ++i)
                if (rows[i] == d && cols[i] == src) {
                    if (first < 0) first = i;
                    ++cnt;
                }
            for (int i = 0; i < nterms; ++i) {
                if (rows[i] < 0 || rows[i] > 3 || cols[i] < 0 || cols[i] > 3)
                    return wl_fail(WL_EINVAL, "term row/column outside 0..3");
                if (rows[i] != d || cols[i] != src) continue;
                ApplyTerm& t = A.t[n++];
                t.dst = static_cast<signed char>(d);
                t.src = static_cast<signed char>(src);
                // the identity shortcut: a diagonal entry that IS the constant 1
                t.one = (d == src && cnt == 1 && km[first] == 0 && kn[first] == 0 &&
                         coeff[first] == 1.0)
                            ? 1 : 0;
                t.pad = 0;
                t.dr = static_cast<short>(-kn[i]);
                t.dc = static_cast<short>(-km[i]);
                t.c = static_cast<float>(coeff[i]);
            }
        }
    }
    A.t0[4] = n;
    A.nterms = n;
    const dim3 block(128), grid((qw + 127) / 128, qh, 4);
    if (qh > 65535) return wl_fail(WL_EINVAL, "apply_step supports up to 65535 plane rows");
    apply_step_kernel<<<grid, block, 0, static_cast<cudaStream_t>(stream)>>>(A);
    wl_count_launch();
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return wl_fail(WL_ERUNTIME, cudaGetErrorString(e));
    return WL_OK;
}

}  // extern "C"
