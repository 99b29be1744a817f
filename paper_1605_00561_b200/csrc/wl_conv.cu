// Direct 2-D convolution forward (SchemeKind::Convolution) for cdf53/cdf97.
//
// The reference evaluates the four 2-D analysis filters F_ss' at subsampled
// positions (transform.cpp:129-152; 64 / 256 taps per quad, schemes.cpp:
// 177-181). This kernel stages a (2*TQY + taps) x (2*TQX + 8) pixel tile in
// shared memory by TMA (border tiles: the out-of-image pixels of the
// zero-filled box are then overwritten with their wrapped/mirrored sources on
// the IMAGE grid, which is exact for a single-pass filter), then each
// thread slides over the input pixel rows of an M x 4 quad block, keeping the
// row segment and the 16*M accumulators in registers. The only block barrier
// is the data-availability one (count_barriers = 1). The taps are
// compile-time constants (gen/conv_gen.cuh), summed filter row by filter row
// with mirror-image pixel pairs added first (row2s) instead of the
// reference's std::map order (tolerance regime; exact for cdf53 on dyadic
// inputs). Two horizontally adjacent quad pairs share one packed FFMA2.
#include <cuda.h>

#include "gen/conv_gen.cuh"
#include "wl_fast_impl.cuh"

namespace {

// Thread block: M quad rows x Q = 4 quads (two packed pairs: quads (0, 2)
// and (1, 3) share every tap, FFMA2 with the coefficient broadcast). The
// thread slides down the 2M + 7 (cdf97) input pixel rows of its block once;
// each staged row is loaded ONCE and feeds every output row whose filter
// window covers it (instead of once per output row), so shared-memory
// traffic per output is ~(2M + 8) / (9M) of the one-row version.
#ifndef WL_CONV_M
#define WL_CONV_M 4  // 2 before the fold; with it 4 rows win (cdf97 0.133 -> 0.129 ms, cdf53 0.102 -> 0.093)
#endif
// Mirror-symmetric filter rows folded (x[c-d] + x[c+d] added once, shared by
// the components with that centre column): 25 instead of 32 FP32 ops per
// quad and input row for cdf97 (row2s), else every tap (row2).
#ifndef WL_CONV_FOLD
#define WL_CONV_FOLD 1
#endif
#ifndef WL_CONV_TQY
#define WL_CONV_TQY 32
#endif
constexpr int TQX = 64, TQY = WL_CONV_TQY, Q = 4, QP = Q / 2, M = WL_CONV_M;
constexpr int NT = (TQX / Q) * (TQY / M);  // threads per CTA
constexpr int MARGIN = 4;                  // staged pixel columns left of the tile
constexpr int SW = 2 * TQX + 2 * MARGIN;   // staged row length (136 px)
static_assert(TQY % M == 0 && NT % 32 == 0, "conv block geometry");

template <class C>
struct ConvGeo {
    static constexpr int kRows = 2 * TQY + (C::kRow1 - C::kRow0);
    static constexpr int kBytes = kRows * SW * 4;
    static constexpr int kSpan = C::kCol1 - C::kCol0;      // taps per row - 1
    static constexpr int kPairs = 2 * (QP - 1) + kSpan + 1;  // packed row segment
    static_assert(C::kCol0 >= -MARGIN && 2 * Q + kSpan + (C::kCol0 + MARGIN) <= 16,
                  "row segment inside the four 16-byte loads");
};

// Image-grid index resolution for border tiles (periodic wrap / whole-point
// mirror, transform.cpp:59-72); one conditional step when the overshoot is
// smaller than the image, the general loop otherwise.
__device__ __forceinline__ int resolve(int i, int n, int boundary) {
    if (i >= 0 && i < n) return i;
    if (n == 1) return 0;
    if (boundary == 0) {
        if (i < 0 && i + n >= 0) return i + n;
        if (i >= n && i - n < n) return i - n;
        int m = i % n;
        return m < 0 ? m + n : m;
    }
    if (i < 0 && -i < n) return -i;
    if (i >= n && 2 * (n - 1) - i >= 0) return 2 * (n - 1) - i;
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
    const bool interior = py0 >= 0 && px0 >= 0 && py0 + G::kRows <= h && px0 + SW <= w;
    if (a.has_map) {
        // every tile through TMA; outside the image the box is zero-filled
        if (threadIdx.x == 0) {
            wlfast::mbar_init(bar, 1);
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
            wlfast::mbar_expect_tx(bar, G::kBytes);
            wlfast::tma_load_3d(px, &m, bar, px0, py0, b);
        }
        __syncthreads();  // barrier init visible before anyone waits on it
        wlfast::mbar_wait(bar, 0);
        if (!interior) {
            // border tile: overwrite the out-of-image pixels with their
            // wrapped / mirrored sources (image grid, exact for one pass);
            // one warp per staged row, whole rows only when the row is outside
            const int xl = px0 < 0 ? -px0 : 0;               // columns [0, xl) outside
            const int xr = px0 + SW > w ? w - px0 : SW;       // columns [xr, SW) outside
            for (int y = threadIdx.x / 32; y < G::kRows; y += NT / 32) {
                const int yy = py0 + y;
                const bool row_out = yy < 0 || yy >= h;
                const float* src = img + (long)resolve(yy, h, a.boundary) * a.in_pitch;
                for (int x = threadIdx.x & 31; x < SW; x += 32)
                    if (row_out || x < xl || x >= xr)
                        px[y * SW + x] = src[resolve(px0 + x, w, a.boundary)];
            }
            __syncthreads();
        }
    } else {
        // no tensor map (unaligned pitch / pointer): element-wise staging
        for (int y = threadIdx.x / 32; y < G::kRows; y += NT / 32) {
            const float* src = img + (long)resolve(py0 + y, h, a.boundary) * a.in_pitch;
            for (int x = threadIdx.x & 31; x < SW; x += 32)
                px[y * SW + x] = src[resolve(px0 + x, w, a.boundary)];
        }
        __syncthreads();  // the single data-availability barrier
    }

    const int qb = threadIdx.x % (TQX / Q), mb = threadIdx.x / (TQX / Q);
    wl2 acc[M][QP][4];
#pragma unroll
    for (int i = 0; i < M; ++i)
#pragma unroll
        for (int p = 0; p < QP; ++p)
#pragma unroll
            for (int c = 0; c < 4; ++c) acc[i][p][c] = 0ull;  // (+0.f, +0.f)
    // staged pixel column of buf[0]: the lane's 2Q own pixels start at 8*qb + MARGIN
    const float* base = px + (2 * M * mb) * SW + 2 * Q * qb;
    constexpr int kOff = C::kCol0 + MARGIN;  // seg[i] = buf[i + kOff]
    wlfast::sfor<2 * (M - 1) + (C::kRow1 - C::kRow0) + 1>([&](auto j_) {
        constexpr int J = decltype(j_)::value;
        const float* row = base + J * SW;
        float buf[16];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const float4 u = reinterpret_cast<const float4*>(row)[k];
            buf[4 * k] = u.x; buf[4 * k + 1] = u.y; buf[4 * k + 2] = u.z; buf[4 * k + 3] = u.w;
        }
        wl2 pr[G::kPairs];
#pragma unroll
        for (int i = 0; i < G::kPairs; ++i) pr[i] = wl_pk_keep(buf[i + kOff], buf[i + kOff + Q]);
        wlfast::sfor<M>([&](auto m_) {
            constexpr int MM = decltype(m_)::value;
            constexpr int Y = J + C::kRow0 - 2 * MM;  // filter row of this input row
            if constexpr (Y >= C::kRow0 && Y <= C::kRow1) {
                if constexpr (WL_CONV_FOLD)
                    C::template row2s<Y, QP>(pr, acc[MM]);
                else
                    C::template row2<Y, QP>(pr, acc[MM]);
            }
        });
    });
    const int gx = c0 + Q * qb;
#pragma unroll
    for (int i = 0; i < M; ++i) {
        const int gy = r0 + M * mb + i;
        if (gy >= a.yhi) break;
        float o[Q][4];
#pragma unroll
        for (int p = 0; p < QP; ++p)
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                o[p][c] = wl_lo(acc[i][p][c]);
                o[p + QP][c] = wl_hi(acc[i][p][c]);
            }
        if (a.scaling) {
#pragma unroll
            for (int q = 0; q < Q; ++q) {
                o[q][0] *= a.scale;
                o[q][3] /= a.scale;
            }
        }
        const long off = (long)(gy - a.ylo) * a.out_pitch + gx;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            float* p = a.out[c] + b * a.out_bstride[c] + off;
            if (a.vec4 && gx + Q <= a.qw) {
                *reinterpret_cast<float4*>(p) = make_float4(o[0][c], o[1][c], o[2][c], o[3][c]);
            } else {
#pragma unroll
                for (int q = 0; q < Q; ++q)
                    if (gx + q < a.qw) p[q] = o[q][c];
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
