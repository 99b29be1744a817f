// Direct 2-D convolution forward (SchemeKind::Convolution) for cdf53/cdf97.
//
// The reference evaluates the four 2-D analysis filters F_ss' at subsampled
// positions (transform.cpp:129-152; 64 / 256 taps per quad, schemes.cpp:
// 177-181). This kernel stages a (2*TQY + taps) x (2*TQX + 8) pixel tile in
// shared memory (TMA for interior tiles; wrapped/mirrored loads on the IMAGE
// grid for border tiles, which is exact for a single-pass filter), then each
// thread slides over the input pixel rows of a 1 x Q quad strip, keeping the
// row segment and the 4*Q accumulators in registers. The only block barrier
// is the data-availability one (count_barriers = 1). The taps are
// compile-time constants (gen/conv_gen.cuh), summed in row-major order
// instead of the reference's std::map order (tolerance regime; exact for
// cdf53 on dyadic inputs).
#include <cuda.h>

#include "gen/conv_gen.cuh"
#include "wl_fast_impl.cuh"

namespace {

#ifndef WL_CONV_Q
#define WL_CONV_Q 4
#endif
// Row segments via lane-swizzled 16-byte loads + shuffles (1) or overlapping
// 8-byte loads (0: 4-way shared-memory bank conflicts). Measured
// (profiles/tuning_r02_conv.txt): cdf53 -10..-14% with shuffles, cdf97
// +14..16% (its 9 rows x 8 shuffles cost more than the conflicts), so the
// shuffle layout serves cdf53 only.
#ifndef WL_CONV_SHFL
#define WL_CONV_SHFL 1
#endif
#ifndef WL_CONV_TQY
#define WL_CONV_TQY 32
#endif
constexpr int TQX = 64, TQY = WL_CONV_TQY, Q = WL_CONV_Q, NT = 256;
constexpr int MARGIN = 4;                 // staged pixel columns left of the tile
constexpr int SW = 2 * TQX + 2 * MARGIN;  // staged row length (136 px)

template <class C>
struct ConvGeo {
    static constexpr int kRows = 2 * TQY + (C::kRow1 - C::kRow0);
    static constexpr int kBytes = kRows * SW * 4;
    static constexpr int kSeg = 2 * Q + (C::kCol1 - C::kCol0);
};

__device__ __forceinline__ int resolve(int i, int n, int boundary) {
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

struct ConvArgs {
    const float* img;
    long in_pitch;
    float* out[4];
    long out_pitch;
    int qw, qh, boundary, scaling;
    float scale;
    int vec4;     // output pitch/pointers allow float4 stores
    int has_map;  // TMA descriptor valid (else every tile takes the LDG path)
    long in_bstride, out_bstride[4];  // batch: elements between images (blockIdx.z)
    int ylo, yhi;                  // stored quad rows [ylo, yhi); out[] addresses row ylo
};

template <class C>
__global__ void __launch_bounds__(NT) conv_fast_kernel(const __grid_constant__ CUtensorMap m,
                                                       const ConvArgs a) {
    using G = ConvGeo<C>;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    float* px = reinterpret_cast<float*>(smem_raw);
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem_raw + G::kBytes);
    const int w = 2 * a.qw, h = 2 * a.qh;
    const int r0 = a.ylo + blockIdx.y * TQY, c0 = blockIdx.x * TQX;
    const int b = blockIdx.z;
    const float* img = a.img + b * a.in_bstride;
    // previous grid complete (PDL launch); no-op otherwise. No early trigger:
    // this grid is not persistent, dependents must not take its SM slots.
    wlfast::pdl_wait();
    const int py0 = 2 * r0 + C::kRow0, px0 = 2 * c0 - MARGIN;
    const bool interior = a.has_map && py0 >= 0 && px0 >= 0 && py0 + G::kRows <= h &&
                          px0 + SW <= w;
    if (interior) {
        if (threadIdx.x == 0) {
            wlfast::mbar_init(bar, 1);
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
            wlfast::mbar_expect_tx(bar, G::kBytes);
            wlfast::tma_load_3d(px, &m, bar, px0, py0, b);
        }
        __syncthreads();  // barrier init visible before anyone waits on it
        wlfast::mbar_wait(bar, 0);
    } else {
        for (int i = threadIdx.x; i < G::kRows * SW; i += NT) {
            const int y = i / SW, x = i - (i / SW) * SW;
            const int ry = resolve(py0 + y, h, a.boundary), rx = resolve(px0 + x, w, a.boundary);
            px[i] = img[(long)ry * a.in_pitch + rx];
        }
        __syncthreads();  // the single data-availability barrier
    }

    constexpr int kBlocksX = TQX / Q;
#pragma unroll
    for (int k = 0; k < (TQY * kBlocksX) / NT; ++k) {
        const int blk = threadIdx.x + k * NT;
        const int qr = blk / kBlocksX, qb = blk - (blk / kBlocksX) * kBlocksX;
        float acc[Q][4];
#pragma unroll
        for (int q = 0; q < Q; ++q)
#pragma unroll
            for (int c = 0; c < 4; ++c) acc[q][c] = 0.f;
        if constexpr (WL_CONV_SHFL && C::kCol1 == 2) {
        // Row segment of the lane's Q quads: its own 2Q pixels with two
        // 16-byte loads in a lane-swizzled order (every 8-lane phase covers
        // all 32 banks: conflict-free), the -kCol0 / kCol1 halo pixels from
        // the neighbour lanes by shuffle (a half-warp spans one 64-quad tile
        // row); only the segment's edge lanes read their halo from memory.
        static_assert(Q == 4 && TQX == 64, "shuffle layout: 16 lanes x 4 quads per row");
        constexpr int HL = -C::kCol0, HR = C::kCol1;
        const int lane = threadIdx.x & 31, sw = (lane >> 2) & 1;
        wlfast::sfor<C::kRow1 - C::kRow0 + 1>([&](auto y_) {
            constexpr int Y = decltype(y_)::value + C::kRow0;
            const float* own = px + (2 * qr + Y - C::kRow0) * SW + MARGIN + 2 * Q * qb;
            const float4 u0 = *reinterpret_cast<const float4*>(own + 4 * sw);
            const float4 u1 = *reinterpret_cast<const float4*>(own + 4 * (sw ^ 1));
            const float4 lo = sw ? u1 : u0, hi = sw ? u0 : u1;
            const float o[8] = {lo.x, lo.y, lo.z, lo.w, hi.x, hi.y, hi.z, hi.w};
            float seg[G::kSeg];
#pragma unroll
            for (int i = 0; i < HL; ++i) seg[i] = __shfl_up_sync(0xffffffffu, o[8 - HL + i], 1, 16);
#pragma unroll
            for (int i = 0; i < 8; ++i) seg[HL + i] = o[i];
#pragma unroll
            for (int i = 0; i < HR; ++i) seg[HL + 8 + i] = __shfl_down_sync(0xffffffffu, o[i], 1, 16);
            if (qb == 0) {
#pragma unroll
                for (int i = 0; i < HL; ++i) seg[i] = own[i - HL];
            }
            if (qb == kBlocksX - 1) {
#pragma unroll
                for (int i = 0; i < HR; ++i) seg[HL + 8 + i] = own[8 + i];
            }
            C::template row<Y, Q>(seg, acc);
        });
        } else {
        // pixel column of seg[0] inside the staged tile
        const int sx = 2 * Q * qb + MARGIN + C::kCol0;
        wlfast::sfor<C::kRow1 - C::kRow0 + 1>([&](auto y_) {
            constexpr int Y = decltype(y_)::value + C::kRow0;
            const float* row = px + (2 * qr + Y - C::kRow0) * SW + sx;
            float seg[G::kSeg];
#pragma unroll
            for (int i = 0; i < G::kSeg; i += 2) {
                const float2 v = *reinterpret_cast<const float2*>(row + i);
                seg[i] = v.x;
                seg[i + 1] = v.y;
            }
            C::template row<Y, Q>(seg, acc);
        });
        }
        const int gy = r0 + qr, gx = c0 + Q * qb;
        if (gy >= a.yhi) continue;
        if (a.scaling) {
#pragma unroll
            for (int q = 0; q < Q; ++q) {
                acc[q][0] *= a.scale;
                acc[q][3] /= a.scale;
            }
        }
        const long off = (long)(gy - a.ylo) * a.out_pitch + gx;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            float* p = a.out[c] + b * a.out_bstride[c] + off;
            if (a.vec4 && gx + Q <= a.qw) {
                static_assert(Q % 4 == 0, "float4 stores of Q quads");
#pragma unroll
                for (int q = 0; q < Q; q += 4)
                    *reinterpret_cast<float4*>(p + q) =
                        make_float4(acc[q][c], acc[q + 1][c], acc[q + 2][c], acc[q + 3][c]);
            } else {
#pragma unroll
                for (int q = 0; q < Q; ++q)
                    if (gx + q < a.qw) p[q] = acc[q][c];
            }
        }
    }
}

template <class C>
cudaError_t launch_conv(const WlLevel& L, cudaStream_t stream) {
    using G = ConvGeo<C>;
    ConvArgs a{};
    a.img = L.in[0];
    a.in_pitch = L.in_pitch;
    for (int k = 0; k < 4; ++k) a.out[k] = L.out[k];
    a.out_pitch = L.out_pitch;
    a.qw = L.qw;
    a.qh = L.qh;
    a.boundary = L.boundary;
    const WlProgram& P = wl_host_program(L.prog);
    a.scaling = L.scaling && P.has_scale;
    a.scale = P.scale;
    bool v4 = (L.out_pitch % 4) == 0;
    for (int k = 0; k < 4; ++k) v4 = v4 && (reinterpret_cast<uintptr_t>(L.out[k]) % 16) == 0;
    for (int k = 0; k < 4; ++k) v4 = v4 && ((L.nb > 1 ? L.out_bstride[k] : 0) % 4) == 0;
    a.vec4 = v4;
    CUtensorMap m{};
    const int nb = L.nb > 1 ? L.nb : 1;
    a.in_bstride = nb > 1 ? L.in_bstride[0] : 0;
    for (int k = 0; k < 4; ++k) a.out_bstride[k] = nb > 1 ? L.out_bstride[k] : 0;
    a.ylo = L.yhi > 0 ? L.ylo : 0;
    a.yhi = L.yhi > 0 ? L.yhi : L.qh;
    a.has_map = wlfast::make_map(&m, L.in[0], 2 * L.qw, 2 * L.qh, L.in_pitch, nb, a.in_bstride,
                                 SW, G::kRows);
    const size_t smem = G::kBytes + 16;
    static bool attr[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (!attr[dev & 63]) {
        cudaFuncSetAttribute(conv_fast_kernel<C>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem);
        attr[dev & 63] = true;
    }
    const dim3 grid((L.qw + TQX - 1) / TQX, (a.yhi - a.ylo + TQY - 1) / TQY, nb);
    cudaError_t le = wlfast::launch_pdl(conv_fast_kernel<C>, grid, dim3(NT), smem, stream, m, a);
    wl_count_launch();
    return le != cudaSuccess ? le : cudaGetLastError();
}

}  // namespace

cudaError_t wl_launch_conv_fast(const WlLevel& L, cudaStream_t stream) {
    if (L.wavelet == 0) return launch_conv<Conv_cdf53>(L, stream);
    if (L.wavelet == 1) return launch_conv<Conv_cdf97>(L, stream);
    return cudaErrorNotSupported;
}
