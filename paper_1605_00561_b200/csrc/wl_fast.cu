// Fast register-tile engine: host side (TMA descriptors, tile plan, frame
// hand-off to the interpreter, dispatch to the per-(wavelet, direction)
// instantiation units wl_fast_<wavelet>_<dir>.cu).
#include <cstdint>
#include <cstdlib>
#include <mutex>
#include <type_traits>

#include "wl_fast_impl.cuh"

namespace wlfast {

// Which (wavelet, direction) launches claim tiles dynamically: bit
// 2 * wavelet + direction (cdf53 fwd 0x1, inv 0x2; cdf97 0x4 / 0x8; dd137
// 0x10 / 0x20). Measured per direction (profiles/tuning_r02_s2.txt, bench on
// one box): the cdf53 forwards and the cdf97 inverses need them at 16384^2
// (0.40 -> 0.32 ms, 0.45 -> 0.33 ms); the one-CTA-per-SM cdf97 forwards are
// 2-3% faster at 8192^2 and in the configs[3] pyramid with static tiles.
#ifndef WL_DYN_DEFAULT_MASK
#define WL_DYN_DEFAULT_MASK 0x3b
#endif

// Dynamic tile-claim counters (FastArgs::sched): one zeroed device ring per
// device; a slot is {claim counter, exit counter} and the last CTA of the
// launch using it resets it to zero. Eager launches cycle through the first
// kEager slots (a slot is reused only after kEager further launches, far
// beyond the launch queue); launches captured into a CUDA graph get a slot of
// their own from the rest, never reused (a replay may run concurrently with
// eager launches); none left -> nullptr (static round robin). WL_DYN=0 turns
// dynamic claims off.
bool dyn_claims(int wavelet, int dir) {
    static const int mask = [] {
        const char* e = getenv("WL_DYN_MASK");
        return e ? (int)strtol(e, nullptr, 0) : WL_DYN_DEFAULT_MASK;
    }();
    return (mask >> (2 * wavelet + dir)) & 1;
}

unsigned* sched_slot(cudaStream_t stream) {
    constexpr int kEager = 4096, kSlots = 8192;
    static std::mutex mu;
    static unsigned* ring[64] = {};
    static int next_eager[64] = {}, next_cap[64] = {};
    static const bool off = [] {
        const char* e = getenv("WL_DYN");
        return e && e[0] == '0';
    }();
    if (off) return nullptr;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev >= 64) return nullptr;
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(stream, &cs) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    std::lock_guard<std::mutex> lk(mu);
    if (!ring[dev]) {
        if (cs != cudaStreamCaptureStatusNone) return nullptr;  // no allocation while capturing
        // relaxed capture mode: a global-mode capture in another thread must
        // not be invalidated by this one-time allocation; zeroed on the
        // (non-capturing) caller stream and waited for there only
        cudaStreamCaptureMode mode = cudaStreamCaptureModeRelaxed;
        cudaThreadExchangeStreamCaptureMode(&mode);
        unsigned* p = nullptr;
        const bool ok = cudaMalloc(&p, sizeof(unsigned) * 2 * kSlots) == cudaSuccess &&
                        cudaMemsetAsync(p, 0, sizeof(unsigned) * 2 * kSlots, stream) == cudaSuccess &&
                        cudaStreamSynchronize(stream) == cudaSuccess;
        cudaThreadExchangeStreamCaptureMode(&mode);
        if (!ok) {
            if (p) cudaFree(p);
            cudaGetLastError();
            return nullptr;
        }
        ring[dev] = p;
    }
    if (cs != cudaStreamCaptureStatusNone) {
        if (kEager + next_cap[dev] >= kSlots) return nullptr;
        return ring[dev] + 2 * (kEager + next_cap[dev]++);
    }
    const int k = next_eager[dev];
    next_eager[dev] = (k + 1) % kEager;
    return ring[dev] + 2 * k;
}

EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q{};
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) !=
                cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            return static_cast<EncodeTiledFn>(nullptr);
        return reinterpret_cast<EncodeTiledFn>(p);
    }();
    return fn;
}

bool make_map(CUtensorMap* m, const float* base, int w, int h, long pitch, int nb, long bstride,
              int box_w, int box_h) {
    EncodeTiledFn enc = encode_fn();
    if (!enc) return false;
    if (nb < 1) nb = 1;
    if (nb == 1) bstride = pitch * static_cast<long>(h);  // any valid stride
    if ((reinterpret_cast<uintptr_t>(base) & 15) || ((pitch * 4) & 15) || ((bstride * 4) & 15))
        return false;
    const cuuint64_t dims[3] = {static_cast<cuuint64_t>(w), static_cast<cuuint64_t>(h),
                                static_cast<cuuint64_t>(nb)};
    const cuuint64_t strides[2] = {static_cast<cuuint64_t>(pitch) * 4,
                                   static_cast<cuuint64_t>(bstride) * 4};
    const cuuint32_t box[3] = {static_cast<cuuint32_t>(box_w), static_cast<cuuint32_t>(box_h), 1};
    const cuuint32_t es[3] = {1, 1, 1};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(base), dims, strides,
               box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
               CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace wlfast

cudaError_t wl_fast_cdf53_fwd(int scheme, const WlLevel& L, const wlfast::Plan& p,
                              cudaStream_t s);
cudaError_t wl_fast_cdf53_inv(int scheme, const WlLevel& L, const wlfast::Plan& p,
                              cudaStream_t s);
cudaError_t wl_fast_cdf97_fwd(int scheme, const WlLevel& L, const wlfast::Plan& p,
                              cudaStream_t s);
cudaError_t wl_fast_cdf97_inv(int scheme, const WlLevel& L, const wlfast::Plan& p,
                              cudaStream_t s);
cudaError_t wl_fast_cdf53_direct(int scheme, const WlLevel& L, const wlfast::Plan& p,
                                 cudaStream_t s);
cudaError_t wl_fast_cdf97_direct(int scheme, const WlLevel& L, const wlfast::Plan& p,
                                 cudaStream_t s);
cudaError_t wl_fast_dd137_fwd(int scheme, const WlLevel& L, const wlfast::Plan& p,
                              cudaStream_t s);
cudaError_t wl_fast_dd137_inv(int scheme, const WlLevel& L, const wlfast::Plan& p,
                              cudaStream_t s);
cudaError_t wl_fast_dd137_direct(int scheme, const WlLevel& L, const wlfast::Plan& p,
                                 cudaStream_t s);
namespace {

template <class C>
void geo(int* R, int* NW, int* CPT, int* KR) {
    *R = C::R;
    *NW = C::NW;
    *CPT = C::CPT;
    *KR = C::KR;
}

// Tile geometry of the instantiation that serves (wavelet, scheme, direction)
// -- must match the SchemeConfig the kernel was compiled with.
template <int W, int D, bool DIRECT, int S>
using CfgOf = std::conditional_t<DIRECT, wlfast::DirectConfigOf<W, D, S>, wlfast::SchemeConfig<W, D, S>>;
template <int W, int D, bool DIRECT>
void geo_wd(int scheme, int* R, int* NW, int* CPT, int* KR) {
    switch (scheme) {
        case 0: return geo<CfgOf<W, D, DIRECT, 0>>(R, NW, CPT, KR);
        case 1: return geo<CfgOf<W, D, DIRECT, 1>>(R, NW, CPT, KR);
        case 2: return geo<CfgOf<W, D, DIRECT, 2>>(R, NW, CPT, KR);
        case 3: return geo<CfgOf<W, D, DIRECT, 3>>(R, NW, CPT, KR);
        case 4: return geo<CfgOf<W, D, DIRECT, 4>>(R, NW, CPT, KR);
        case 5: return geo<CfgOf<W, D, DIRECT, 5>>(R, NW, CPT, KR);
        case 6: return geo<CfgOf<W, D, DIRECT, 6>>(R, NW, CPT, KR);
        case 7: return geo<CfgOf<W, D, DIRECT, 7>>(R, NW, CPT, KR);
        default: return geo<CfgOf<W, D, DIRECT, 8>>(R, NW, CPT, KR);
    }
}

// Tile geometry of the instantiation that serves L (TMA or direct-load).
template <bool DIRECT>
void geometry_of(const WlLevel& L, int* R, int* NW, int* CPT, int* KR) {
    const bool f = L.direction == 0;
    if (L.wavelet == 0)
        f ? geo_wd<0, 0, DIRECT>(L.scheme, R, NW, CPT, KR) : geo_wd<0, 1, DIRECT>(L.scheme, R, NW, CPT, KR);
    else if (L.wavelet == 1)
        f ? geo_wd<1, 0, DIRECT>(L.scheme, R, NW, CPT, KR) : geo_wd<1, 1, DIRECT>(L.scheme, R, NW, CPT, KR);
    else
        f ? geo_wd<2, 0, DIRECT>(L.scheme, R, NW, CPT, KR) : geo_wd<2, 1, DIRECT>(L.scheme, R, NW, CPT, KR);
}
void geometry(const WlLevel& L, int* R, int* NW, int* CPT, int* KR) {
    geometry_of<false>(L, R, NW, CPT, KR);
}

// Programs the fast engine serves: cdf53 / cdf97 lifting schemes, and the
// dd137 lifting schemes except Polyphase(*) (reach 3, interpreter).
bool fast_program(int wavelet, int scheme) {
    if (wavelet < 0 || wavelet > 2 || scheme < 0 || scheme > 8) return false;
    return wavelet < 2 || scheme <= 6;
}

bool aligned(const void* p, int bytes) { return (reinterpret_cast<uintptr_t>(p) % bytes) == 0; }

}  // namespace

namespace {

// The TMA path: 16-byte aligned boxes and pitches (tensor maps), and for
// CPT = 4 the aligned float4 stores (plane widths and pitches in multiples
// of 4 cells).
bool tma_ok(const WlLevel& L, int CPT) {
    if (!wlfast::encode_fn()) return false;
    if (L.direction == 0) {
        if (!aligned(L.in[0], 16) || (L.in_pitch % 4) != 0) return false;
        for (int k = 0; k < 4; ++k)
            if (!aligned(L.out[k], 8)) return false;
        if (L.out_pitch % 2 != 0) return false;
    } else {
        for (int k = 0; k < 4; ++k)
            if (!aligned(L.in[k], 16)) return false;
        if ((L.in_pitch % 4) != 0 || !aligned(L.out[0], 16) || (L.out_pitch % 4) != 0)
            return false;
    }
    if (L.nb > 1)
        for (int k = 0; k < 4; ++k)
            if ((L.in_bstride[k] % 4) != 0 || (L.out_bstride[k] % 4) != 0) return false;
    if (CPT == 4) {
        if (L.qw % 4 != 0 || L.out_pitch % 4 != 0) return false;
        for (int k = 0; k < (L.direction == 0 ? 4 : 1); ++k)
            if (!aligned(L.out[k], 16) || (L.nb > 1 && L.out_bstride[k] % 4 != 0)) return false;
    }
    return true;
}

// The direct-load path: float2 loads of pixel pairs (forward), scalar
// everything else; no halo wait (the strip runtime then waits in its
// exchange kernel).
bool direct_ok(const WlLevel& L) {
    if (L.xflag_a) return false;
    if (L.direction == 0) {  // float2 loads of pixel pairs: every row 8-byte aligned
        if (!aligned(L.in[0], 8) || L.in_pitch % 2 != 0) return false;
        if (L.nb > 1 && L.in_bstride[0] % 2 != 0) return false;
    }
    for (int k = 0; k < 4; ++k)
        if ((L.in[k] && !aligned(L.in[k], 4)) || (L.out[k] && !aligned(L.out[k], 4))) return false;
    return true;
}

}  // namespace

int wl_fast_mode(const WlLevel& L) {
    if (!fast_program(L.wavelet, L.scheme)) return 0;
    int R, NW, CPT, KR;
    geometry(L, &R, &NW, &CPT, &KR);
    const int H = wl_host_program(L.prog).halo;
    const bool force_direct = wl_engine() == 3;
    if (!force_direct && tma_ok(L, CPT) && wlfast::plan_tiles(L, H, R, NW, CPT, false, false, KR).ok)
        return 1;
    geometry_of<true>(L, &R, &NW, &CPT, &KR);
    if (direct_ok(L) && wlfast::plan_tiles(L, H, R, NW, CPT, true, false, KR).ok) return 2;
    return 0;
}

bool wl_fast_supported(const WlLevel& L) { return wl_fast_mode(L) != 0; }

cudaError_t wl_launch_fast(const WlLevel& L, cudaStream_t stream) {
    const int mode = wl_fast_mode(L);
    if (!mode) return cudaErrorNotSupported;
    int R, NW, CPT, KR;
    if (mode == 2)
        geometry_of<true>(L, &R, &NW, &CPT, &KR);
    else
        geometry(L, &R, &NW, &CPT, &KR);
    const int H = wl_host_program(L.prog).halo;
    const wlfast::Plan plan = wlfast::plan_tiles(L, H, R, NW, CPT, mode == 2, false, KR);
    cudaError_t e;
    if (mode == 2)
        e = L.wavelet == 0   ? wl_fast_cdf53_direct(L.scheme, L, plan, stream)
            : L.wavelet == 1 ? wl_fast_cdf97_direct(L.scheme, L, plan, stream)
                             : wl_fast_dd137_direct(L.scheme, L, plan, stream);
    else if (L.wavelet == 0)
        e = L.direction == 0 ? wl_fast_cdf53_fwd(L.scheme, L, plan, stream)
                             : wl_fast_cdf53_inv(L.scheme, L, plan, stream);
    else if (L.wavelet == 1)
        e = L.direction == 0 ? wl_fast_cdf97_fwd(L.scheme, L, plan, stream)
                             : wl_fast_cdf97_inv(L.scheme, L, plan, stream);
    else
        e = L.direction == 0 ? wl_fast_dd137_fwd(L.scheme, L, plan, stream)
                             : wl_fast_dd137_inv(L.scheme, L, plan, stream);
    if (e != cudaSuccess) return e;
    // periodic, or symmetric with mirrored border tiles: the grid covers the image
    if (plan.args.wrap || plan.args.mirror) return cudaSuccess;
    // Symmetric: the frame around the tile grid (image borders included) goes
    // to the interpreter, which mirrors every out-of-image read per step.
    const int Y0 = plan.args.Y0, X0 = plan.args.X0;
    const int Y1 = Y0 + plan.tiles_y * plan.args.TH, X1 = X0 + plan.args.tiles_x * plan.args.TW;
    WlRects fr{};
    fr.n = 4;
    fr.y0[0] = 0;  fr.x0[0] = 0;  fr.ny[0] = Y0;          fr.nx[0] = L.qw;       // top
    fr.y0[1] = Y1; fr.x0[1] = 0;  fr.ny[1] = L.qh - Y1;   fr.nx[1] = L.qw;       // bottom
    fr.y0[2] = Y0; fr.x0[2] = 0;  fr.ny[2] = Y1 - Y0;     fr.nx[2] = X0;         // left
    fr.y0[3] = Y0; fr.x0[3] = X1; fr.ny[3] = Y1 - Y0;     fr.nx[3] = L.qw - X1;  // right
    // symmetric window: only the stored rows [ylo, yhi) of the frame, into
    // outputs addressed from the window's first row
    const int wy0 = L.yhi > 0 ? L.ylo : 0, wy1 = L.yhi > 0 ? L.yhi : L.qh;
    for (int k = 0; k < 4; ++k) {
        const int a = fr.y0[k] > wy0 ? fr.y0[k] : wy0;
        const int b = fr.y0[k] + fr.ny[k] < wy1 ? fr.y0[k] + fr.ny[k] : wy1;
        fr.y0[k] = a;
        fr.ny[k] = b > a ? b - a : 0;
    }
    const int nb = L.nb > 1 ? L.nb : 1;
    for (int b = 0; b < nb; ++b) {  // the frame of every image of a batch
        WlLevel Li = L;
        Li.nb = 1;
        Li.ylo = Li.yhi = 0;
        for (int k = 0; k < 4; ++k) {
            if (Li.in[k]) Li.in[k] += b * L.in_bstride[k];
            if (Li.out[k]) Li.out[k] += b * L.out_bstride[k];
            // row 0 of the virtual whole plane (never written outside [wy0, wy1))
            if (Li.out[k] && wy0) Li.out[k] -= static_cast<long>(wy0) * L.out_pitch *
                                               (L.direction == 0 ? 1 : 2);
        }
        e = wl_launch_interp_rects(Li, fr, stream);
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}
