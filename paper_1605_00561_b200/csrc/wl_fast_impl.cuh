// Fast register-tile engine for the cdf53 / cdf97 lifting schemes.
//
// Persistent CTAs; warp-specialised:
//   * 1 producer warp streams tiles HBM -> shared memory with TMA
//     (cp.async.bulk.tensor.3d) into an NS-stage ring guarded by mbarriers
//     ("full": transaction-count barrier armed with the stage's bytes;
//     "empty": one arrival per compute warp once it has copied its rows).
//   * NW compute warps hold the tile in registers: warp w owns R rows of
//     component cells, lane l owns CPT=2 adjacent cells of each row, i.e. a
//     64-cell-wide x (NW*R)-cell-tall compute region per tile. The 2x2 pixel
//     de-interleave of polyphase_split (transform.cpp:74-86) happens in the
//     LDS.128 of two pixel rows.
//   * Every lifting step runs on registers. Horizontal neighbours come from
//     the adjacent lane by warp shuffle; vertical neighbours from the same
//     lane's registers, except at the warp's top/bottom row, where they come
//     from the neighbouring warp through shared memory. That exchange is the
//     ONLY cross-warp dependency, so each tile executes exactly one
//     bar.sync per epoch after the first (whose neighbour rows are read
//     straight from the TMA stage, behind the mbarrier wait): block
//     barriers per tile == count_barriers of the scheme (schemes.cpp:193-198).
//   * Redundant halo: the outer H cells of the compute region (H = the
//     program's reach, = parsim required_halo) are computed but not stored;
//     output tile = (64 - 2H) x (NW*R - 2H) cells.
//
// Only tiles whose compute region (plus one ghost row above and below) lies
// inside the image are processed here; they are identical for the periodic
// and symmetric boundaries. The thin frame outside the tile grid is handled
// by the generic interpreter (wl_interp.cu), which implements the per-step
// boundary resolution of transform.cpp:114-115 exactly.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <type_traits>
#include <utility>

#include "gen/fast_gen.cuh"
#include "wl_internal.h"

namespace wlfast {

// Producer wait on a released stage: test_wait + __nanosleep back-off (cap
// per program, ProdBackoff). try_wait with a suspend hint or a plain try_wait
// loop measured 10-40% slower (their polling competes with the compute warps).
// Tuning knobs: pad the exchange buffer to at least this many component rows
// (shared-memory footprint / residency experiments) and cap CTAs per SM
// (0 = as many as fit).
#ifndef WL_XCH_MIN
#define WL_XCH_MIN 0
#endif
#ifndef WL_PROD_EARLY
#define WL_PROD_EARLY 0
#endif
#ifndef WL_PROD_BO97_FWD  // the cdf97 forwards on the long cap too (A/B knob)
#define WL_PROD_BO97_FWD 0
#endif
#ifndef WL_PROD_BACKOFF97_NS
#define WL_PROD_BACKOFF97_NS 1024
#endif
#ifndef WL_PROD_BACKOFF_NS
#define WL_PROD_BACKOFF_NS 256
#endif


// CPT = component cells per lane per row (2 or 4); the compute region is
// 32 * CPT cells wide. CPT = 4 stores one aligned float4 per lane and plane
// and keeps tile boundaries on 32-byte sectors.
// Horizontal halo of the stored columns: CPT = 2 uses the program's reach H;
// CPT = 4 drops whole lanes (HX = 4 cells, lanes 0 and 31).
template <int CPT, int H>
constexpr int halo_x() { return CPT == 4 ? 4 : H; }

template <class F, int... I>
__device__ __forceinline__ void sfor_impl(F&& f, std::integer_sequence<int, I...>) {
    (f(std::integral_constant<int, I>{}), ...);
}
template <int N, class F>
__device__ __forceinline__ void sfor(F&& f) {
    sfor_impl(f, std::make_integer_sequence<int, N>{});
}

__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WL_WAIT:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WL_WAIT;\n}" ::"r"(smem_u32(b)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar,
                                            int x, int y) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_u32(bar))
        : "memory");
}
// 3-D box (x, y, image of a batch).
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar,
                                            int x, int y, int z) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
        : "memory");
}
// Producer-side wait: the TMA warp is normally far ahead of the compute
// warps, so poll with exponential back-off instead of a tight spin that
// steals issue slots from the compute warps sharing its scheduler.
__device__ __forceinline__ bool mbar_test(uint64_t* b, unsigned parity) {
    unsigned ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n}"
        : "=r"(ok)
        : "r"(smem_u32(b)), "r"(parity)
        : "memory");
    return ok != 0;
}
template <int CAP = WL_PROD_BACKOFF_NS>
__device__ __forceinline__ void mbar_wait_backoff(uint64_t* b, unsigned parity) {
    unsigned ns = 32;
    while (!mbar_test(b, parity)) {
        __nanosleep(ns);
        ns = ns < CAP ? 2 * ns : CAP;
    }
}
#ifndef WL_CLAIM_LATE
#define WL_CLAIM_LATE 0
#endif
#ifndef WL_RAMP1
#define WL_RAMP1 0
#endif
// Direct-load (unaligned) forwards: realigned float4 stores (1) or
// element-wise stores (0); WL_REALIGN97 extends them to cdf97. With 3-row warps
// (WL_DIRECT_R = 3) every lifting forward gains (8190^2: cdf53 -8..-16%, cdf97
// -6..-16%) except the Polyphase ones, which keep element-wise stores (and
// 4-row warps for cdf97), and the reach-2 dd137 kernels (+8..10%)
// (profiles/tuning_r02_s2.txt, tools/ab_runs/g6, g7, g10, g16).
#ifndef WL_REALIGN_STORES
#define WL_REALIGN_STORES 1
#endif
#ifndef WL_REALIGN97
#define WL_REALIGN97 1
#endif
// Direct-load inverses: float2 / float4 image-row stores (1) or element-wise (0).
// Measured at 8190^2 / 8194^2: -4..-14% for every CPT = 2 inverse except the
// cdf53 Polyphase(*) ones (+1..+7%, kept element-wise) (tools/ab_runs/g8_invpair.sh);
// the CPT = 4 cdf97 Polyphase inverse 0.373 -> 0.234 ms (g13_inv4.sh).
#ifndef WL_INV_PAIR_STORES
#define WL_INV_PAIR_STORES 1
#endif
// A/B knobs: border tiles of periodic plans from the TMA box + wrapped
// re-reads of the outside cells (1) or every cell from global memory (0);
// periodic grid from cell 0 with clamped last row/column (1) or the former
// grid with a tile row/column before the image (0).
#ifndef WL_BORDER_TMA
#define WL_BORDER_TMA 1
#endif
#ifndef WL_PLAN_V2
#define WL_PLAN_V2 1
#endif
// Forward input tile as WL_FWD_SPLIT TMA boxes of 2*kRows/WL_FWD_SPLIT rows.
#ifndef WL_FWD_SPLIT
#define WL_FWD_SPLIT 1
#endif
#ifndef WL_LDS_SWIZZLE
#define WL_LDS_SWIZZLE 1
#endif
#ifndef WL_WRAP_MOD_INV
#define WL_WRAP_MOD_INV 1
#endif
#ifndef WL_SYM_FAST
#define WL_SYM_FAST 1
#endif
#ifndef WL_STORE_PAIRS
#define WL_STORE_PAIRS 0
#endif

// Programmatic dependent launch: wait until the preceding grid in the stream
// has completed and its writes are visible (no-op for normal launches), and
// let the next PDL-launched grid get scheduled while this one drains.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
#ifndef WL_PDL
#define WL_PDL 0  // measured 3.7% slower on the bench step (profiles/tuning_r01_pdl.txt)
#endif

// Launch with the programmatic-stream-serialization attribute (PDL).
template <class K, class... Args>
cudaError_t launch_pdl(K kern, dim3 grid, dim3 block, size_t smem, cudaStream_t stream,
                       Args... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = WL_PDL;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, args...);
}

__device__ __forceinline__ void named_sync(int id, int nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

struct FastArgs {
    const float* in[4];  // fwd: in[0] = image; inv: LL, HL, LH, HH (wrapped border loads)
    long in_pitch;
    float* out[4];       // fwd: LL, HL, LH, HH planes; inv: out[0] = image
    long out_pitch;      // elements
    int qw, qh;          // component-grid size
    int tiles_x, ntiles; // ntiles = images x tiles per image
    int ntiles_img;      // tiles per image
    int tx0, ty0;        // index of the first tile column / row (-1 when covering borders)
    int X0, Y0;          // first output cell of tile (0, 0)
    int xlast, ylast;    // tile origins clamped to these (last tile column / row
                         // ends at the image edge, overlapping its neighbour)
    int TW, TH;          // output tile size in cells
    int wrap;            // periodic plan covering the whole image (border tiles wrap)
    int scaling;
    float scale;
    long in_bstride[4], out_bstride[4];  // per plane: elements between images of a batch
    int ylo, yhi;        // stored cell rows [ylo, yhi); out[] addresses row ylo
    int mirror;          // symmetric plan covering the whole image (border tiles mirror)
    int filter;          // 0 every tile, 1 interior tiles only, 2 border tiles only
    // strip halo wait (WlLevel::xflag_a): edge tile rows last, producer waits
    const unsigned* xflag_a;
    const unsigned* xflag_b;
    unsigned xepoch;
    unsigned* xerr;
    // dynamic tile claims: {claim counter, exit counter}, zero at launch and
    // reset by the last CTA to exit (wl_sched_slot); null = static round robin
    unsigned* sched;
    // WL_DIAG_TIMES builds only: per CTA {entry, first tile ready, exit, tiles}
    // (%globaltimer ns), wl_diag_set(); null otherwise
    unsigned long long* diag;
};

// Tile-row order: with a halo wait the window's first and last tile rows go
// last (sequence k -> row: 1..n-2, 0, n-1), so the wait overlaps the
// interior tiles. (Row n-2 can also reach the lower halo when the last row
// is short; it then simply waits a little earlier.)
__device__ __forceinline__ int tile_row_of(int k, int n, bool edge_last) {
    if (!edge_last || n <= 2) return k;
    return k < n - 2 ? k + 1 : (k == n - 2 ? 0 : n - 1);
}

// System-scope acquire spin on two flags (halo pushed by neighbour ranks),
// bounded by a 10 s timeout that sets *err.
__device__ __forceinline__ unsigned ld_acquire_sys_u32(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
static __device__ __noinline__ void wait_halo_flags(const unsigned* fa, const unsigned* fb, unsigned e,
                                             unsigned* err) {
    unsigned long long t0, t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    unsigned ns = 64;
    while ((int)(ld_acquire_sys_u32(fa) - e) < 0 || (int)(ld_acquire_sys_u32(fb) - e) < 0) {
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        if (t - t0 > 10ull * 1000 * 1000 * 1000) {
            atomicExch(err, 1u);
            return;
        }
        __nanosleep(ns);
        ns = ns < 1024 ? 2 * ns : 1024;
    }
    // the halo rows will be read by TMA (async proxy) and generic loads
    asm volatile("fence.proxy.async.global;" ::: "memory");
}

// Kernel arguments: one level per launch (lv[0]).
struct KArgs {
    FastArgs lv[1];
};

__device__ __host__ __forceinline__ int floordiv(int a, int b) {
    return a >= 0 ? a / b : -((-a + b - 1) / b);
}
// First stored cell column / row of tile column tx / row ty (grid indices
// already offset by tx0 / ty0).
__device__ __forceinline__ int tile_xs(const FastArgs& a, int tx) {
    const int x = a.X0 + tx * a.TW;
    return x < a.xlast ? x : a.xlast;
}
__device__ __forceinline__ int tile_ys(const FastArgs& a, int ty) {
    const int y = a.Y0 + ty * a.TH;
    return y < a.ylast ? y : a.ylast;
}
__device__ __forceinline__ unsigned ld_relaxed_gpu_u32(const unsigned* p) {
    unsigned v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
// Producer back-off cap (ns) per program: the polling producer shares an SM
// sub-partition with compute warps, so how long it sleeps between polls is
// a trade-off between refill latency and stolen issue slots. Measured on
// B200 at 16384^2 (profiles/tuning_r01_backoff.txt): 1024 ns for the cdf97
// lifting inverses (+6-13%; two CTAs of 4 compute warps per SM share the
// sub-partitions with the producers), 256 ns elsewhere (cdf53 inverses and
// the FP32-heavy cdf97 Polyphase inverse lose with the longer cap; the
// forwards are neutral within noise).
template <class P, int DIR>
struct ProdBackoff {
    static constexpr int ns = P::kHalo == 2 && (DIR == 1 || WL_PROD_BO97_FWD)
                                  ? WL_PROD_BACKOFF97_NS
                                  : WL_PROD_BACKOFF_NS;
};
template <>
struct ProdBackoff<P_cdf97_polyphase_inv, 1> {
    static constexpr int ns = WL_PROD_BACKOFF_NS;
};

template <int R, int NW, int CPT, int NS = 2, int NXC = 4, int KR = 1>
struct Geometry {
    static constexpr int kStages = NS;                       // TMA ring depth
    static constexpr int TWC = 32 * CPT;                     // compute-region width in cells
    static constexpr int kRows = NW * R + 2 * KR;            // cell rows per stage incl. KR ghosts
    static constexpr int kStageFloats = 4 * TWC * kRows;     // == 2*TWC px * 2*kRows px
    static constexpr int kStageBytes = kStageFloats * 4;
    // edge exchange: 2 slots x NW warps x NXC published component rows of
    // 32 * CPT cells (NXC = the most component rows any epoch reads across warps)
    static constexpr int kXchFloats = 2 * NW * (NXC > WL_XCH_MIN ? NXC : WL_XCH_MIN) * 32 * CPT;
    static constexpr size_t kSmemBytes =
        NS * (size_t)kStageBytes + (size_t)kXchFloats * 4 + 16 * NS;
    // CTAs per SM the shared memory allows (228 KB per SM, 1 KB reserved per CTA)
    static constexpr int kMinBlocks = 2 * (kSmemBytes + 1024) <= 233472 ? 2 : 1;
};

// Neighbour accessor for the cell at (row RR, column CC) of the lane's block:
// KR ghost rows above (gu[0] = row -KR) and below (gd[0] = row R), and per
// block row KR cells left (sl[.][j] = column -1-j) / right (sr[.][j] = column
// CPT+j) from the adjacent lanes; sl/sr rows are indexed block row + KR.
template <int R, int CPT, int KR, int RR, int CC>
struct Acc {
    const float (&v)[R][CPT][4];
    const float (&gu)[KR][CPT][4];
    const float (&gd)[KR][CPT][4];
    const float (&sl)[R + 2 * KR][KR][4];
    const float (&sr)[R + 2 * KR][KR][4];
    template <int C, int DR, int DC>
    __device__ __forceinline__ float g() const {
        constexpr int r = RR + DR, c = CC + DC;
        if constexpr (c < 0)
            return sl[r + KR][-c - 1][C];
        else if constexpr (c >= CPT)
            return sr[r + KR][c - CPT][C];
        else if constexpr (r < 0)
            return gu[r + KR][c][C];
        else if constexpr (r >= R)
            return gd[r - R][c][C];
        else
            return v[r][c][C];
    }
};

// Pair mode (FP32-issue-bound programs, CPT = 4): the lane's four cells of a
// row are held as two packed pairs A = (c0, c2), B = (c1, c3) and every tap
// of P::nbr2 is ONE packed FFMA2 for two cells (same per-cell operation
// sequence as the scalar code). Horizontal neighbours of a pair are the
// pairs L = (c-1, c1) and Rt = (c2, c4) (c-1 / c4 from the adjacent lanes),
// built once per row and epoch. Output pair PP (0 = A, 1 = B) of block row
// RR reads position k = PP + DC in {L, A, B, Rt} of block row RR + DR
// (-1 = the ghost row above, R = below); lt / rt hold L / Rt per block row.
template <int R, int RR, int PP>
struct AccP {
    const wl2 (&v2)[R][2][4];
    const wl2 (&gu2)[2][4];
    const wl2 (&gd2)[2][4];
    const wl2 (&lt)[R + 2][4];
    const wl2 (&rt)[R + 2][4];
    template <int C, int DR, int DC>
    __device__ __forceinline__ wl2 g() const {
        constexpr int r = RR + DR, k = PP + DC;
        if constexpr (k < 0)
            return lt[r + 1][C];
        else if constexpr (k > 1)
            return rt[r + 1][C];
        else if constexpr (r < 0)
            return gu2[k][C];
        else if constexpr (r >= R)
            return gd2[k][C];
        else
            return v2[r][k][C];
    }
};
// Programs that may run in pair mode: the cdf97 Polyphase forward and inverse
// (126 MACs per cell in two neighbour epochs, no local steps). Measured OFF
// (profiles/tuning_r02_s2.txt): 24% fewer instructions, but 4% slower at
// 8192^2 (0.165 vs 0.158 ms; stalls move to fixed-latency dependencies of
// the half as many, twice as wide accumulation chains) -- the kernel is not
// issue-bound. WL_PAIR_POLY=1 turns it on (A/B knob).
#ifndef WL_PAIR_POLY
#define WL_PAIR_POLY 0
#endif
template <class P>
struct PairMode {
    static constexpr bool on = false;
};
template <>
struct PairMode<P_cdf97_polyphase_fwd> {
    static constexpr bool on = WL_PAIR_POLY;
};
template <>
struct PairMode<P_cdf97_polyphase_inv> {
    static constexpr bool on = WL_PAIR_POLY;
};

// Neighbour reads of one epoch (gen_steps.py usage_masks): per source
// component c, bit (dr + k) * (2k + 1) + (dc + k) for every tap offset, k =
// the program's reach (P::kReach: 1 for cdf53 / cdf97, 2 for dd137).
struct UseT {
    unsigned long long m[4];
    int k;
};
template <class P, int E>
__host__ __device__ constexpr UseT use_of() {
    return UseT{{P::kUse[E][0], P::kUse[E][1], P::kUse[E][2], P::kUse[E][3]}, P::kReach};
}
__host__ __device__ constexpr bool uses(const UseT& u, int c, int dr, int dc) {
    if (dr < -u.k || dr > u.k || dc < -u.k || dc > u.k) return false;
    return (u.m[c] >> ((dr + u.k) * (2 * u.k + 1) + (dc + u.k))) & 1ull;
}
__host__ __device__ constexpr bool uses_dc(const UseT& u, int c, int dc) {
    for (int dr = -u.k; dr <= u.k; ++dr)
        if (uses(u, c, dr, dc)) return true;
    return false;
}
__host__ __device__ constexpr bool uses_dr(const UseT& u, int c, int dr) {
    for (int dc = -u.k; dc <= u.k; ++dc)
        if (uses(u, c, dr, dc)) return true;
    return false;
}
// Is cell (block row r, lane-relative column c) of component C read by any
// of the lane's R x CPT cells? (r in [-k, R + k), c in [-k, CPT + k))
__host__ __device__ constexpr bool reads(const UseT& u, int C, int r, int c, int R, int CPT) {
    for (int t = 0; t < R; ++t)
        for (int cc = 0; cc < CPT; ++cc)
            if (uses(u, C, r - t, c - cc)) return true;
    return false;
}
// Exchange mode: minimal (publish only the component rows the neighbour
// warps read this epoch: a lifting epoch reads across warps from one side
// only, 2 components; Polyphase up to 6) or full (the k edge rows on both
// sides, all 4 components). Chosen per configuration by measurement
// (Config::XF). xch_up / xch_dn = rows of component c published for the warp
// below / above: rows R-1..R-n / 0..n-1 of this warp, n = the deepest read.
__host__ __device__ constexpr int xch_up(const UseT& u, int c, bool full) {
    if (full) return u.k;
    for (int n = u.k; n >= 1; --n)
        if (uses_dr(u, c, -n)) return n;
    return 0;
}
__host__ __device__ constexpr int xch_dn(const UseT& u, int c, bool full) {
    if (full) return u.k;
    for (int n = u.k; n >= 1; --n)
        if (uses_dr(u, c, n)) return n;
    return 0;
}
__host__ __device__ constexpr int xch_rank(const UseT& u, int c, int dr, bool full) {
    int n = 0;
    for (int k = 0; k < c; ++k) n += dr < 0 ? xch_up(u, k, full) : xch_dn(u, k, full);
    return n;
}
__host__ __device__ constexpr int xch_count(const UseT& u, int dr, bool full) {
    return xch_rank(u, 4, dr, full);
}
// The same queries through a tag type carrying the epoch's UseT as a static
// member (usable inside the nested per-component lambdas of the kernel,
// where a captured constexpr struct is not a constant expression).
template <class P, int E>
struct UseOf {
    static constexpr UseT u = use_of<P, E>();
};
template <class UO, class = decltype(UO::u)>
__host__ __device__ constexpr bool uses(UO, int c, int dr, int dc) { return uses(UO::u, c, dr, dc); }
template <class UO, class = decltype(UO::u)>
__host__ __device__ constexpr bool uses_dc(UO, int c, int dc) { return uses_dc(UO::u, c, dc); }
template <class UO, class = decltype(UO::u)>
__host__ __device__ constexpr bool uses_dr(UO, int c, int dr) { return uses_dr(UO::u, c, dr); }
template <class UO, class = decltype(UO::u)>
__host__ __device__ constexpr bool reads(UO, int C, int r, int c, int R, int CPT) {
    return reads(UO::u, C, r, c, R, CPT);
}
template <class UO, class = decltype(UO::u)>
__host__ __device__ constexpr int xch_up(UO, int c, bool full) { return xch_up(UO::u, c, full); }
template <class UO, class = decltype(UO::u)>
__host__ __device__ constexpr int xch_dn(UO, int c, bool full) { return xch_dn(UO::u, c, full); }
template <class UO, class = decltype(UO::u)>
__host__ __device__ constexpr int xch_rank(UO, int c, int dr, bool full) {
    return xch_rank(UO::u, c, dr, full);
}
template <class UO, class = decltype(UO::u)>
__host__ __device__ constexpr int xch_count(UO, int dr, bool full) { return xch_count(UO::u, dr, full); }

template <class P, bool FULL, int E = 1>
constexpr int xch_comps() {
    if constexpr (E >= P::kEpochs) {
        return 0;
    } else {
        constexpr UseT u = use_of<P, E>();
        constexpr int n = xch_count(u, -1, FULL) + xch_count(u, 1, FULL);
        constexpr int rest = xch_comps<P, FULL, E + 1>();
        return n > rest ? n : rest;
    }
}

// Direct-load variant: no stage ring (shared memory holds only the edge
// exchange), so its occupancy is set by registers: shorter warp rows
// (WL_DIRECT_R, at least 2 x reach; DirectConfig) and WL_DIRECT_MINB CTAs per
// SM let a second CTA's loads overlap the first one's compute.
#ifndef WL_DIRECT_NW
#define WL_DIRECT_NW 8
#endif
#ifndef WL_DIRECT_R
#define WL_DIRECT_R 3  // 4 before the realigned stores (tools/ab_runs/g10_direct97.sh)
#endif
#ifndef WL_DIRECT_MINB
#define WL_DIRECT_MINB 2
#endif
template <class P>
struct DirectMinBlocks {  // reach-2 rows and the 126-MAC cdf97 Polyphase epochs need
    static constexpr int value = P::kReach > 1 ? 1 : WL_DIRECT_MINB;  // their registers
};
template <>
struct DirectMinBlocks<P_cdf97_polyphase_fwd> {
    static constexpr int value = 1;
};
template <>
struct DirectMinBlocks<P_cdf97_polyphase_inv> {
    static constexpr int value = 1;
};

// DIRECT: no TMA -- shapes whose pitches/pointers/widths the TMA boxes and
// the aligned float4 stores cannot take (e.g. 8190^2 images: 32760-byte rows,
// odd plane widths). Every tile loads its cells with coalesced per-lane
// global loads (the periodic border-tile path) and stores element by element
// under a column mask; the producer warp exits at once and the stage ring is
// not allocated. Same instruction sequence per cell, so the same results.
template <class P, int DIR, int R, int NW, int CPT, int NS, bool XF, bool MIRROR,
          bool DIRECT = false>
__global__ void __launch_bounds__((NW + 1) * 32,
                                  (DIRECT ? DirectMinBlocks<P>::value
                                          : Geometry<R, NW, CPT, NS, xch_comps<P, XF>(), P::kReach>::kMinBlocks))
    fast_kernel(const __grid_constant__ CUtensorMap m0, const __grid_constant__ CUtensorMap m1,
                const __grid_constant__ CUtensorMap m2, const __grid_constant__ CUtensorMap m3,
                const __grid_constant__ KArgs K) {
    static_assert(!DIRECT || !MIRROR, "direct-load launches: plain plans");
    __shared__ int4 task_sm[NS];  // dynamic claims: the tile of each stage (producer -> consumers)
    constexpr int NXC = xch_comps<P, XF>();
    constexpr int KR = P::kReach;  // ghost rows / neighbour cells a step reads
    static_assert(R >= 2 * KR && KR <= CPT, "edge rows / lane-neighbour cells");
    static_assert(KR == 1 || !MIRROR, "reach-2 programs: plain / direct plans");
    using G = Geometry<R, NW, CPT, NS, NXC, KR>;
    constexpr int H = P::kHalo;
    constexpr int TWC = G::TWC;
    constexpr int HX = halo_x<CPT, H>();
    extern __shared__ __align__(128) unsigned char smem_raw[];
    float* stage = reinterpret_cast<float*>(smem_raw);
    float* xch = stage + (DIRECT ? 0 : NS * G::kStageFloats);
    uint64_t* full = reinterpret_cast<uint64_t*>(xch + G::kXchFloats);
    uint64_t* empty = full + NS;

    const FastArgs& a = K.lv[0];  // per-tile code rebinds it to the tile's level
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#ifdef WL_DIAG_TIMES
    auto gtime = [] {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        return t;
    };
    unsigned long long* dg = a.diag ? a.diag + 4 * blockIdx.x : nullptr;
    if (dg && threadIdx.x == 0) dg[0] = gtime();
    int diag_tiles = 0;
#endif
    if (threadIdx.x == 0) {
        for (int k = 0; k < NS; ++k) {
            mbar_init(&full[k], 1);
            mbar_init(&empty[k], NW * 32);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    // everything above touched shared memory only: overlap it with the
    // previous kernel's tail, then order all global traffic after it
    pdl_wait();
    pdl_trigger();

    if (warp == NW) {
        // ---------------- producer warp: TMA tile stream ----------------
        if constexpr (DIRECT) return;  // compute warps load their own cells
        if (lane == 0 && a.sched) {
            // Dynamic tile claims: the first tile is blockIdx.x, every further
            // one comes from a global counter, so CTAs on SMs that run ahead
            // take more tiles and the launch's tail shrinks (static round robin
            // left 7-20 us between the first and the last CTA to finish at
            // 8192^2, tools/diag_times.py). The tile index goes to the compute
            // warps through task_sm; -1 ends their loop.
            // WL_CLAIM_LATE: claim the next tile only once a stage is free (a CTA
            // then holds at most NS tiles, not NS + 1, when the counter runs
            // out -- a shorter tail), paying the atomic's round trip before the
            // load instead of overlapping it.
            bool halo_ready = false;
            int t = blockIdx.x;
            for (int i = 0;; ++i) {
                const int s = i % NS;
                const unsigned use = i / NS;
                if (WL_CLAIM_LATE) {
                    if (i >= NS) mbar_wait_backoff<ProdBackoff<P, DIR>::ns>(&empty[s], (use - 1) & 1);
                    if (i > 0) t = gridDim.x + (int)atomicAdd(a.sched, 1u);
                }
                if (a.filter) {  // interior-only / border-only launch of a symmetric plan
                    for (; t < a.ntiles; t = gridDim.x + (int)atomicAdd(a.sched, 1u)) {
                        const int fb = t / a.ntiles_img, ft = t - fb * a.ntiles_img;
                        const int fy = ft / a.tiles_x;
                        const int fx0 = tile_xs(a, ft - fy * a.tiles_x + a.tx0) - HX;
                        const int fy0 = tile_ys(a, fy + a.ty0) - H - KR;
                        const bool bd = fx0 < 0 || fy0 < 0 || fx0 + TWC > a.qw || fy0 + G::kRows > a.qh;
                        if (bd == (a.filter == 2)) break;
                    }
                }
                if (!WL_CLAIM_LATE && i >= NS)
                    mbar_wait_backoff<ProdBackoff<P, DIR>::ns>(&empty[s], (use - 1) & 1);
                if (t >= a.ntiles) {
                    task_sm[s] = make_int4(-1, 0, 0, 0);
                    mbar_arrive(&full[s]);  // consumers see the sentinel and stop
                    break;
                }
                task_sm[s] = make_int4(t, 0, 0, 0);
                const int b = t / a.ntiles_img, tt = t - b * a.ntiles_img;
                const int tyk = tt / a.tiles_x;
                const int tyi = a.xflag_a ? tile_row_of(tyk, a.ntiles_img / a.tiles_x, true) : tyk;
                const int ty = tyi + a.ty0, tx = tt - tyk * a.tiles_x + a.tx0;
                const int cx = tile_xs(a, tx) - HX;
                const int cy = tile_ys(a, ty) - H - KR;
                if (a.xflag_a && !halo_ready && (cy < a.ylo || cy + G::kRows > a.yhi)) {
                    wait_halo_flags(a.xflag_a, a.xflag_b, a.xepoch, a.xerr);
                    halo_ready = true;
                }
                float* dst = stage + s * G::kStageFloats;
                // WL_RAMP1: the second tile's box only after the first one landed
                // (the first tiles of all CTAs do not share HBM with the second ones)
                if (WL_RAMP1 && i == 1) mbar_wait_backoff<64>(&full[0], 0);
                mbar_expect_tx(&full[s], G::kStageBytes);
                if (DIR == 0) {
                    constexpr int kSplitRows = 2 * G::kRows / WL_FWD_SPLIT;
#pragma unroll
                    for (int q = 0; q < WL_FWD_SPLIT; ++q)
                        tma_load_3d(dst + q * kSplitRows * 2 * TWC, &m0, &full[s], 2 * cx,
                                    2 * cy + q * kSplitRows, b);
                } else {
                    constexpr int plane = TWC * G::kRows;
                    tma_load_3d(dst, &m0, &full[s], cx, cy, b);
                    tma_load_3d(dst + plane, &m1, &full[s], cx, cy, b);
                    tma_load_3d(dst + 2 * plane, &m2, &full[s], cx, cy, b);
                    tma_load_3d(dst + 3 * plane, &m3, &full[s], cx, cy, b);
                }
                if (!WL_CLAIM_LATE) t = gridDim.x + (int)atomicAdd(a.sched, 1u);  // overlaps the load
            }
            // the last producer out resets the slot for the next launch using it
            // (every producer's final claim precedes its exit count)
            if (atomicAdd(a.sched + 1, 1u) == gridDim.x - 1) {
                a.sched[0] = 0;
                a.sched[1] = 0;
            }
        } else if (lane == 0) {
            bool halo_ready = false;
            for (int i = 0, t = blockIdx.x; t < a.ntiles; t += gridDim.x) {
                if (a.filter) {  // interior-only / border-only launch of a symmetric plan
                    const int fb = t / a.ntiles_img, ft = t - fb * a.ntiles_img;
                    const int fy = ft / a.tiles_x;
                    const int fx0 = tile_xs(a, ft - fy * a.tiles_x + a.tx0) - HX;
                    const int fy0 = tile_ys(a, fy + a.ty0) - H - KR;
                    const bool bd = fx0 < 0 || fy0 < 0 || fx0 + TWC > a.qw || fy0 + G::kRows > a.qh;
                    if (bd != (a.filter == 2)) continue;
                }
                const int s = i % NS;
                const unsigned use = i / NS;  // how often stage s was filled before
#if !WL_PROD_EARLY
                if (i >= NS) mbar_wait_backoff<ProdBackoff<P, DIR>::ns>(&empty[s], (use - 1) & 1);
#endif
                const int b = t / a.ntiles_img, tt = t - b * a.ntiles_img;
                const int tyk = tt / a.tiles_x;
                const int tyi = a.xflag_a ? tile_row_of(tyk, a.ntiles_img / a.tiles_x, true) : tyk;
                const int ty = tyi + a.ty0, tx = tt - tyk * a.tiles_x + a.tx0;
                const int cx = tile_xs(a, tx) - HX;     // first compute cell column
                const int cy = tile_ys(a, ty) - H - KR;  // ghost row above the region
                if (a.xflag_a && !halo_ready && (cy < a.ylo || cy + G::kRows > a.yhi)) {
                    wait_halo_flags(a.xflag_a, a.xflag_b, a.xepoch, a.xerr);
                    halo_ready = true;
                }
#if WL_PROD_EARLY  // tile coordinates first: their divisions overlap the stage wait
                if (i >= NS) mbar_wait_backoff<ProdBackoff<P, DIR>::ns>(&empty[s], (use - 1) & 1);
#endif
                float* dst = stage + s * G::kStageFloats;
                // WL_RAMP1: the second tile's box only after the first one landed
                // (the first tiles of all CTAs do not share HBM with the second ones)
                if (WL_RAMP1 && i == 1) mbar_wait_backoff<64>(&full[0], 0);
                mbar_expect_tx(&full[s], G::kStageBytes);
                if (DIR == 0) {
                    constexpr int kSplitRows = 2 * G::kRows / WL_FWD_SPLIT;
#pragma unroll
                    for (int q = 0; q < WL_FWD_SPLIT; ++q)
                        tma_load_3d(dst + q * kSplitRows * 2 * TWC, &m0, &full[s], 2 * cx,
                                    2 * cy + q * kSplitRows, b);
                } else {
                    constexpr int plane = TWC * G::kRows;
                    tma_load_3d(dst, &m0, &full[s], cx, cy, b);
                    tma_load_3d(dst + plane, &m1, &full[s], cx, cy, b);
                    tma_load_3d(dst + 2 * plane, &m2, &full[s], cx, cy, b);
                    tma_load_3d(dst + 3 * plane, &m3, &full[s], cx, cy, b);
                }
                ++i;
            }
        }
        return;
    }

    // ---------------- compute warps ----------------
    float v[R][CPT][4];
    float gu[KR][CPT][4], gd[KR][CPT][4];  // KR ghost rows above / below
    int xslot = 0;

    for (int i = 0, t = blockIdx.x;; t += gridDim.x) {
        const int s = i % NS;
        int b, tyi, txi;
        {
            const FastArgs& a0 = K.lv[0];
            if (!DIRECT && a0.sched) {  // dynamic claims: the producer names the tile
                mbar_wait(&full[s], (i / NS) & 1);
                t = task_sm[s].x;
                if (t < 0) break;
            }
            if (t >= a0.ntiles) break;
            b = t / a0.ntiles_img;
            const int tt = t - b * a0.ntiles_img;
            const int tyk = tt / a0.tiles_x;
            tyi = a0.xflag_a ? tile_row_of(tyk, a0.ntiles_img / a0.tiles_x, true) : tyk;
            txi = tt - tyk * a0.tiles_x;
        }
        // The tile body, instantiated per level with compile-time offsets into
        // K.lv[] (a register-indexed parameter load stalls like a memory load).
        auto body = [&](auto L_) {
            const FastArgs& a = K.lv[decltype(L_)::value];
            const int ty = tyi + a.ty0, tx = txi + a.tx0;
            const int cx = tile_xs(a, tx) - HX;     // first compute cell column
            const int cy = tile_ys(a, ty) - H - KR;  // ghost row above the region
            // Border tile: its compute region leaves the image. Periodic plans
            // load its cells with wrapped coordinates straight from global memory
            // (load-time wrap is exact for the periodic extension).
            const bool border = cx < 0 || cy < 0 || cx + TWC > a.qw || cy + G::kRows > a.qh;
            if (a.filter && border != (a.filter == 2)) return;  // the other launch's tile
            const unsigned phase = (i / NS) & 1;  // fill count of stage s (processed tiles)
            ++i;
            // DIRECT: every tile loads from global memory (coordinates wrapped,
            // which is the identity inside the image)
            const bool wrap_tile = DIRECT || (a.wrap && border);
            // Symmetric border tile: out-of-image cells come zero-filled from the
            // TMA box and are never read as such -- before every neighbour step
            // the distance-1 ghosts are overwritten with their mirror images.
            const bool mtile = MIRROR && a.mirror && border;
            const int gy0m = cy + KR + warp * R;  // image row of v[0]
            if constexpr (!DIRECT)
                if (!a.sched) mbar_wait(&full[s], phase);  // (dynamic: waited for the task)
#ifdef WL_DIAG_TIMES
            if (dg && threadIdx.x == 0 && diag_tiles++ == 0) dg[1] = gtime();
#endif
            const float* st = stage + s * G::kStageFloats;

            // Load the warp's rows (+ one ghost row above and below) and split
            // the 2x2 polyphase components.
            // periodic wrap: one conditional add/subtract unless the image is
            // smaller than a tile (then the general modulo)
            const bool small = WL_WRAP_MOD_INV && DIR == 1 || a.qw < TWC || a.qh < G::kRows;
            auto wrapi = [small](int i, int n) {
                if (small) {
                    i %= n;
                    return i < 0 ? i + n : i;
                }
                return i < 0 ? i + n : (i >= n ? i - n : i);
            };
            // one cell (image cell row ry, column rx, already wrapped) from global memory
            auto load_cell = [&](int ry, int rx, float (&c4)[4]) {
                if (DIR == 0) {
                    const float* p =
                        a.in[0] + b * a.in_bstride[0] + (long)(2 * ry) * a.in_pitch + 2 * rx;
                    const float2 u0 = *reinterpret_cast<const float2*>(p);
                    const float2 u1 = *reinterpret_cast<const float2*>(p + a.in_pitch);
                    c4[0] = u0.x;
                    c4[1] = u0.y;
                    c4[2] = u1.x;
                    c4[3] = u1.y;
                } else {
#pragma unroll
                    for (int c = 0; c < 4; ++c)
                        c4[c] = a.in[c][b * a.in_bstride[c] + (long)ry * a.in_pitch + rx];
                }
            };
            // Load the warp's rows (+ one ghost row above and below) and split
            // the 2x2 polyphase components.
            auto load_row = [&](int q, float (&dst)[CPT][4]) {
                // q: cell row in the stage (0 = ghost row above the region)
                if (DIRECT || (!WL_BORDER_TMA && wrap_tile)) {
                    const int ry = wrapi(cy + q, a.qh);
#pragma unroll
                    for (int j = 0; j < CPT; ++j) load_cell(ry, wrapi(cx + CPT * lane + j, a.qw), dst[j]);
                    return;
                }
                if (DIR == 0) {
                    // pixel rows 2q (LL HL LL HL ...) and 2q+1 (LH HH ...)
                    const float* p0 = st + (2 * q) * (2 * TWC) + 2 * CPT * lane;
                    float4 e[CPT / 2], o[CPT / 2];
                    if constexpr (CPT == 4) {
                        // lanes 32 B apart: read the two 16-B halves in an order
                        // swizzled by lane group so every 8-lane phase covers all
                        // 32 banks (no 2-way conflict), then undo the swap
#if WL_LDS_SWIZZLE
                        const int sw = (lane >> 2) & 1;
                        const float4 e0 = *reinterpret_cast<const float4*>(p0 + 4 * sw);
                        const float4 e1 = *reinterpret_cast<const float4*>(p0 + 4 * (sw ^ 1));
                        const float4 o0 = *reinterpret_cast<const float4*>(p0 + 2 * TWC + 4 * sw);
                        const float4 o1 = *reinterpret_cast<const float4*>(p0 + 2 * TWC + 4 * (sw ^ 1));
                        e[0] = sw ? e1 : e0;
                        e[1] = sw ? e0 : e1;
                        o[0] = sw ? o1 : o0;
                        o[1] = sw ? o0 : o1;
#else
                        e[0] = *reinterpret_cast<const float4*>(p0);
                        e[1] = *reinterpret_cast<const float4*>(p0 + 4);
                        o[0] = *reinterpret_cast<const float4*>(p0 + 2 * TWC);
                        o[1] = *reinterpret_cast<const float4*>(p0 + 2 * TWC + 4);
#endif
                    } else {
                        e[0] = *reinterpret_cast<const float4*>(p0);
                        o[0] = *reinterpret_cast<const float4*>(p0 + 2 * TWC);
                    }
#pragma unroll
                    for (int jj = 0; jj < CPT / 2; ++jj) {
                        dst[2 * jj][0] = e[jj].x; dst[2 * jj][1] = e[jj].y;
                        dst[2 * jj][2] = o[jj].x; dst[2 * jj][3] = o[jj].y;
                        dst[2 * jj + 1][0] = e[jj].z; dst[2 * jj + 1][1] = e[jj].w;
                        dst[2 * jj + 1][2] = o[jj].z; dst[2 * jj + 1][3] = o[jj].w;
                    }
                } else {
                    constexpr int plane = TWC * G::kRows;
#pragma unroll
                    for (int c = 0; c < 4; ++c) {
                        const float* p = st + c * plane + q * TWC + CPT * lane;
                        if constexpr (CPT == 4) {
                            const float4 u = *reinterpret_cast<const float4*>(p);
                            dst[0][c] = u.x; dst[1][c] = u.y; dst[2][c] = u.z; dst[3][c] = u.w;
                        } else {
                            const float2 u = *reinterpret_cast<const float2*>(p);
                            dst[0][c] = u.x;
                            dst[1][c] = u.y;
                        }
                    }
                }
                if (WL_BORDER_TMA && wrap_tile) {
                    // Border tile of a periodic plan: the TMA box is zero-filled
                    // outside the image; only those cells are re-read from their
                    // wrapped positions (exact for the periodic extension). The
                    // row test is warp-uniform; columns diverge on edge lanes only.
                    const int yq = cy + q;
                    const bool row_in = yq >= 0 && yq < a.qh;
                    const int ry = row_in ? yq : wrapi(yq, a.qh);
#pragma unroll
                    for (int j = 0; j < CPT; ++j) {
                        const int xq = cx + CPT * lane + j;
                        if (!row_in || xq < 0 || xq >= a.qw) load_cell(ry, wrapi(xq, a.qw), dst[j]);
                    }
                }
            };
#pragma unroll
            for (int k = 0; k < KR; ++k) load_row(warp * R + k, gu[k]);
#pragma unroll
            for (int r = 0; r < R; ++r) load_row(warp * R + KR + r, v[r]);
#pragma unroll
            for (int k = 0; k < KR; ++k) load_row(warp * R + KR + R + k, gd[k]);
            // Release the stage: every lane's own loads are ordered before its
            // arrive (release semantics; a single elected arrive after __syncwarp
            // let the next TMA overwrite rows other lanes had not finished
            // reading), and the proxy fence orders these generic-proxy reads
            // before the async-proxy (TMA) writes of the refill.
            if constexpr (!DIRECT) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                mbar_arrive(&empty[s]);
            }

            if (DIR == 1 && a.scaling) {  // undo scaling first (transform.cpp:180)
#pragma unroll
                for (int c = 0; c < CPT; ++c) {
#pragma unroll
                    for (int k = 0; k < KR; ++k) {
                        gu[k][c][0] *= a.scale; gu[k][c][3] /= a.scale;
                        gd[k][c][0] *= a.scale; gd[k][c][3] /= a.scale;
                    }
#pragma unroll
                    for (int r = 0; r < R; ++r) { v[r][c][0] *= a.scale; v[r][c][3] /= a.scale; }
                }
            }
#pragma unroll
            for (int c = 0; c < CPT; ++c) {
#pragma unroll
                for (int k = 0; k < KR; ++k) {
                    P::pre(gu[k][c]);
                    P::pre(gd[k][c]);
                }
#pragma unroll
                for (int r = 0; r < R; ++r) P::pre(v[r][c]);
            }

            // pair mode: the state as packed pairs A = (c0, c2), B = (c1, c3)
            constexpr bool PM = PairMode<P>::on && CPT == 4 && !MIRROR && KR == 1;
            wl2 v2[PM ? R : 1][2][4], gu2[2][4], gd2[2][4];
            if constexpr (PM) {
                auto pack = [&](const float (&src)[CPT][4], wl2 (&dst)[2][4]) {
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        dst[0][k] = wl_pk_keep(src[0][k], src[2][k]);
                        dst[1][k] = wl_pk_keep(src[1][k], src[3][k]);
                    }
                };
                pack(gu[0], gu2);
                pack(gd[KR - 1], gd2);
#pragma unroll
                for (int r = 0; r < R; ++r) pack(v[r], v2[r < (PM ? R : 1) ? r : 0]);
            }

#ifndef WL_DIAG_NO_COMPUTE
            sfor<P::kEpochs>([&](auto e_) {
                constexpr int E = decltype(e_)::value;
                using UO = UseOf<P, E>;  // this epoch's neighbour reads (UO{} at the queries)
                // Split-phase block barrier for epochs > 0: publish the edge rows
                // and ARRIVE, compute the rows that need no neighbour-warp data,
                // then WAIT and finish the two edge rows. Still exactly one
                // barrier (one mbarrier phase) per epoch per tile.
                // Layout [slot][warp][top|bottom][column c][lane] float4: every
                // warp-wide access is a contiguous 512 B run (4 wavefronts).
                // Published component rows of this epoch: the warp's bottom row for
                // the components the warp below reads from its row above (UP), then
                // its top row for those the warp above reads from below (DN). Each
                // row is [lane] x CPT floats: one contiguous warp-wide access.
                constexpr int NUP = xch_count(UO{}, -1, XF), NDN = xch_count(UO{}, 1, XF);
                constexpr int kCompF = 32 * CPT;
                constexpr int kSlotF = NXC * kCompF;
                float* xw = xch + (xslot * NW + warp) * kSlotF;
                auto put = [&](float* dst, const float (&row)[CPT][4], int C) {
                    if constexpr (CPT == 4)
                        reinterpret_cast<float4*>(dst)[lane] =
                            make_float4(row[0][C], row[1][C], row[2][C], row[3][C]);
                    else
                        reinterpret_cast<float2*>(dst)[lane] = make_float2(row[0][C], row[1][C]);
                };
                auto get = [&](const float* src, float (&row)[CPT][4], int C) {
                    if constexpr (CPT == 4) {
                        const float4 q = reinterpret_cast<const float4*>(src)[lane];
                        row[0][C] = q.x; row[1][C] = q.y; row[2][C] = q.z; row[3][C] = q.w;
                    } else {
                        const float2 q = reinterpret_cast<const float2*>(src)[lane];
                        row[0][C] = q.x; row[1][C] = q.y;
                    }
                };
                if constexpr (PM) {
                    // ---- pair mode: exchange, then rows top to bottom with a
                    // sliding window of L / Rt pairs (one output row's delay
                    // before it replaces its input row)
                    if constexpr (E > 0) {
                        sfor<4>([&](auto c_) {
                            constexpr int C = decltype(c_)::value;
                            if constexpr (xch_up(UO{}, C, XF))
                                reinterpret_cast<ulonglong2*>(xw + xch_rank(UO{}, C, -1, XF) * kCompF)[lane] =
                                    make_ulonglong2(v2[R - 1][0][C], v2[R - 1][1][C]);
                            if constexpr (xch_dn(UO{}, C, XF))
                                reinterpret_cast<ulonglong2*>(xw + (NUP + xch_rank(UO{}, C, 1, XF)) * kCompF)[lane] =
                                    make_ulonglong2(v2[0][0][C], v2[0][1][C]);
                        });
                        named_sync(1, NW * 32);  // the epoch's block barrier
                        sfor<4>([&](auto c_) {
                            constexpr int C = decltype(c_)::value;
                            if constexpr (xch_up(UO{}, C, XF))
                                if (warp > 0) {
                                    const ulonglong2 q = reinterpret_cast<const ulonglong2*>(
                                        xw - kSlotF + xch_rank(UO{}, C, -1, XF) * kCompF)[lane];
                                    gu2[0][C] = q.x;
                                    gu2[1][C] = q.y;
                                }
                            if constexpr (xch_dn(UO{}, C, XF))
                                if (warp < NW - 1) {
                                    const ulonglong2 q = reinterpret_cast<const ulonglong2*>(
                                        xw + kSlotF + (NUP + xch_rank(UO{}, C, 1, XF)) * kCompF)[lane];
                                    gd2[0][C] = q.x;
                                    gd2[1][C] = q.y;
                                }
                        });
                        xslot ^= 1;
                    }
                    wl2 lt[R + 2][4], rt[R + 2][4];
                    // L / Rt pairs of block row T - 1 (0 = ghost row above)
                    auto lr = [&](auto t_) {
                        constexpr int T = decltype(t_)::value - 1;
                        const wl2 (&rw)[2][4] =
                            T < 0 ? gu2 : (T >= R ? gd2 : v2[T < 0 ? 0 : (T >= R ? R - 1 : T)]);
                        sfor<4>([&](auto c_) {
                            constexpr int C = decltype(c_)::value;
                            constexpr bool nl = T < 0 ? uses(UO{}, C, -1, -1)
                                                      : (T >= R ? uses(UO{}, C, 1, -1) : uses_dc(UO{}, C, -1));
                            constexpr bool nr = T < 0 ? uses(UO{}, C, -1, 1)
                                                      : (T >= R ? uses(UO{}, C, 1, 1) : uses_dc(UO{}, C, 1));
                            if constexpr (nl) {
                                const float c3 = __shfl_up_sync(0xffffffffu, wl_hi(rw[1][C]), 1);
                                lt[T + 1][C] = wl_pk_keep(c3, wl_lo(rw[1][C]));
                            }
                            if constexpr (nr) {
                                const float c4 = __shfl_down_sync(0xffffffffu, wl_lo(rw[0][C]), 1);
                                rt[T + 1][C] = wl_pk_keep(wl_hi(rw[0][C]), c4);
                            }
                        });
                    };
                    wl2 o2[R][2][4];
                    lr(std::integral_constant<int, 0>{});
                    lr(std::integral_constant<int, 1>{});
                    sfor<R>([&](auto r_) {
                        constexpr int RR = decltype(r_)::value;
                        lr(std::integral_constant<int, RR + 2>{});
                        sfor<2>([&](auto p_) {
                            AccP<R, RR, decltype(p_)::value> acc{v2, gu2, gd2, lt, rt};
                            P::template nbr2<E>(acc, o2[RR][decltype(p_)::value]);
                        });
                        if constexpr (RR >= 1) {
#pragma unroll
                            for (int k = 0; k < 4; ++k) {
                                v2[RR - 1][0][k] = o2[RR - 1][0][k];
                                v2[RR - 1][1][k] = o2[RR - 1][1][k];
                            }
                        }
                    });
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        v2[R - 1][0][k] = o2[R - 1][0][k];
                        v2[R - 1][1][k] = o2[R - 1][1][k];
                    }
                    (void)NDN;
                    return;
                }
                if constexpr (E > 0) {
                    sfor<4>([&](auto c_) {
                        constexpr int C = decltype(c_)::value;
                        // rows R-1..R-n for the warp below, 0..n-1 for the warp above
#pragma unroll
                        for (int k = 0; k < xch_up(UO{}, C, XF); ++k)
                            put(xw + (xch_rank(UO{}, C, -1, XF) + k) * kCompF, v[R - 1 - k], C);
#pragma unroll
                        for (int k = 0; k < xch_dn(UO{}, C, XF); ++k)
                            put(xw + (NUP + xch_rank(UO{}, C, 1, XF) + k) * kCompF, v[k], C);
                    });
#ifdef WL_BREAK_BARRIER
                    // negative control (acceptance.cpp:283-296 / parsim break_barrier):
                    // drop the barrier of epoch WL_BREAK_BARRIER; racecheck must flag it
                    if constexpr (E != WL_BREAK_BARRIER)
#endif
                    named_sync(1, NW * 32);  // the epoch's block barrier
                }
                // Symmetric border tiles (MIRROR kernel): whole-point mirroring on
                // the component grid, per step (transform.cpp:66-71, 114-115).
                // Every step reads at most one cell away, so before the step the
                // distance-1 ghosts that in-image cells read are overwritten with
                // their mirror images: row -1 := row 1, row qh := row qh-2,
                // column -1 := column 1, column qw := column qw-2 (corners via
                // both). The host picks the grid's row offset so that the source
                // rows always lie in the warp's own registers (plan_tiles).
                // vrow(T): block row T in [-1, R] (gu, v[0..R-1], gd).
                auto vfix = [&](auto gdgu) {  // gdgu: false -> targets in v, true -> gu/gd
                    if (!mtile) return;
                    const int t_top = -gy0m - 1;  // block row holding image row -1
                    const int t_bot = a.qh - gy0m;  // block row holding image row qh
                    sfor<R + 2>([&](auto k_) {
                        constexpr int T = decltype(k_)::value - 1;
                        constexpr bool edge = T < 0 || T >= R;
                        if constexpr (edge == decltype(gdgu)::value) {
                            float (&dst)[CPT][4] = T < 0 ? gu[0] : (T >= R ? gd[0] : v[T < 0 ? 0 : (T >= R ? R - 1 : T)]);
                            if constexpr (T + 2 <= R - 1) {
                                if (T == t_top)
                                    sfor<4>([&](auto c_) {
                                        constexpr int C = decltype(c_)::value;
                                        if constexpr (uses_dr(UO{}, C, -1))
#pragma unroll
                                            for (int c = 0; c < CPT; ++c) dst[c][C] = v[T + 2][c][C];
                                    });
                            }
                            if constexpr (T - 2 >= 0) {
                                if (T == t_bot)
                                    sfor<4>([&](auto c_) {
                                        constexpr int C = decltype(c_)::value;
                                        if constexpr (uses_dr(UO{}, C, 1))
#pragma unroll
                                            for (int c = 0; c < CPT; ++c) dst[c][C] = v[T - 2][c][C];
                                    });
                            }
                        }
                    });
                };
                // horizontal: the lane whose first cell is column 0 reads its left
                // neighbour as its own column 1; the lane whose last cell is column
                // qw-1 reads its right neighbour as its own column qw-2 (cx and qw
                // are multiples of CPT).
                auto hfix = [&](float (&sl_)[R + 2 * KR][KR][4], float (&sr_)[R + 2 * KR][KR][4], int r_lo,
                                int r_hi) {
                    if (!mtile) return;
                    const int gxl = cx + CPT * lane;
                    const bool left = gxl == 0, right = gxl + CPT - 1 == a.qw - 1;
#pragma unroll
                    for (int r = 0; r < R + 2; ++r) {
                        if (r < r_lo || r > r_hi) continue;
                        const float (&src)[CPT][4] =
                            r == 0 ? gu[0] : (r == R + 1 ? gd[0] : v[r == 0 ? 0 : (r > R ? R - 1 : r - 1)]);
                        sfor<4>([&](auto c_) {
                            constexpr int C = decltype(c_)::value;
                            if constexpr (uses_dc(UO{}, C, -1))
                                if (left) sl_[r][0][C] = src[1][C];
                            if constexpr (uses_dc(UO{}, C, 1))
                                if (right) sr_[r][0][C] = src[CPT - 2][C];
                        });
                    }
                };
                if constexpr (MIRROR) vfix(std::false_type{});
                // Horizontal neighbours of the lane's edge columns (warp shuffle).
                float sl[R + 2 * KR][KR][4], sr[R + 2 * KR][KR][4];
                sfor<4>([&](auto c_) {
                    constexpr int C = decltype(c_)::value;
                    sfor<KR>([&](auto j_) {
                        constexpr int J = decltype(j_)::value;  // column -1-J / CPT+J
                        sfor<R>([&](auto r_) {
                            constexpr int r = decltype(r_)::value;
                            if constexpr (reads(UO{}, C, r, -1 - J, R, CPT))
                                sl[r + KR][J][C] = __shfl_up_sync(0xffffffffu, v[r][CPT - 1 - J][C], 1);
                            if constexpr (reads(UO{}, C, r, CPT + J, R, CPT))
                                sr[r + KR][J][C] = __shfl_down_sync(0xffffffffu, v[r][J][C], 1);
                        });
                    });
                });
                if constexpr (MIRROR) hfix(sl, sr, 1, R);
                float o[R][CPT][4];
                auto row = [&](auto r_) {
                    constexpr int RR = decltype(r_)::value;
                    sfor<CPT>([&](auto c_) {
                        constexpr int CC = decltype(c_)::value;
                        Acc<R, CPT, KR, RR, CC> acc{v, gu, gd, sl, sr};
                        P::template nbr<E>(acc, o[RR][CC]);
                    });
                };
                // interior rows KR..R-1-KR read only this warp's rows
                sfor<R - 2 * KR>([&](auto r_) { row(std::integral_constant<int, decltype(r_)::value + KR>{}); });
                if constexpr (E > 0) {
                    sfor<4>([&](auto c_) {
                        constexpr int C = decltype(c_)::value;
                        // bottom rows of the warp above -> gu[KR-1-k], top rows of the
                        // warp below -> gd[k]
#pragma unroll
                        for (int k = 0; k < xch_up(UO{}, C, XF); ++k)
                            if (warp > 0)
                                get(xw - kSlotF + (xch_rank(UO{}, C, -1, XF) + k) * kCompF, gu[KR - 1 - k], C);
#pragma unroll
                        for (int k = 0; k < xch_dn(UO{}, C, XF); ++k)
                            if (warp < NW - 1)
                                get(xw + kSlotF + (NUP + xch_rank(UO{}, C, 1, XF) + k) * kCompF, gd[k], C);
                    });
                    (void)NDN;
                    xslot ^= 1;
                }
                if constexpr (MIRROR) vfix(std::true_type{});
                // lane-neighbour cells of the ghost rows (corners of the stencil)
                sfor<4>([&](auto c_) {
                    constexpr int C = decltype(c_)::value;
                    sfor<KR>([&](auto j_) {
                        constexpr int J = decltype(j_)::value;
                        sfor<KR>([&](auto k_) {
                            constexpr int k = decltype(k_)::value;
                            if constexpr (reads(UO{}, C, k - KR, -1 - J, R, CPT))
                                sl[k][J][C] = __shfl_up_sync(0xffffffffu, gu[k][CPT - 1 - J][C], 1);
                            if constexpr (reads(UO{}, C, R + k, -1 - J, R, CPT))
                                sl[R + KR + k][J][C] = __shfl_up_sync(0xffffffffu, gd[k][CPT - 1 - J][C], 1);
                            if constexpr (reads(UO{}, C, k - KR, CPT + J, R, CPT))
                                sr[k][J][C] = __shfl_down_sync(0xffffffffu, gu[k][J][C], 1);
                            if constexpr (reads(UO{}, C, R + k, CPT + J, R, CPT))
                                sr[R + KR + k][J][C] = __shfl_down_sync(0xffffffffu, gd[k][J][C], 1);
                        });
                    });
                });
                if constexpr (MIRROR) hfix(sl, sr, 0, R + 1);  // corners (and rows again)
                sfor<KR>([&](auto k_) {
                    row(std::integral_constant<int, decltype(k_)::value>{});
                    row(std::integral_constant<int, R - KR + decltype(k_)::value>{});
                });
#pragma unroll
                for (int r = 0; r < R; ++r)
#pragma unroll
                    for (int c = 0; c < CPT; ++c) {
#pragma unroll
                        for (int k = 0; k < 4; ++k) v[r][c][k] = o[r][c][k];
                        P::template post<E>(v[r][c]);
                    }
            });

            if constexpr (PM) {
#pragma unroll
                for (int r = 0; r < R; ++r)
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        v[r][0][k] = wl_lo(v2[r < (PM ? R : 1) ? r : 0][0][k]);
                        v[r][2][k] = wl_hi(v2[r < (PM ? R : 1) ? r : 0][0][k]);
                        v[r][1][k] = wl_lo(v2[r < (PM ? R : 1) ? r : 0][1][k]);
                        v[r][3][k] = wl_hi(v2[r < (PM ? R : 1) ? r : 0][1][k]);
                    }
            }
#endif  // WL_DIAG_NO_COMPUTE
            // ---------------- store ----------------
            const int gy0 = cy + KR + warp * R;  // global cell row of v[0]
            const int gx = cx + CPT * lane;     // global cell col of column 0
            if (DIR == 0 && a.scaling) {  // scale_planes (transform.cpp:154-159)
#pragma unroll
                for (int r = 0; r < R; ++r)
#pragma unroll
                    for (int c = 0; c < CPT; ++c) {
                        v[r][c][0] *= a.scale;
                        v[r][c][3] /= a.scale;
                    }
            }
            // 64-bit row pointers of the lane's first cell, advanced per row
            float* pk[4];
            const long off0 = DIR == 0 ? (long)(gy0 - a.ylo) * a.out_pitch + gx
                                       : (long)(2 * (gy0 - a.ylo)) * a.out_pitch + 2 * gx;
#pragma unroll
            for (int k = 0; k < (DIR == 0 ? 4 : 1); ++k) pk[k] = a.out[k] + b * a.out_bstride[k] + off0;
            const long step = DIR == 0 ? a.out_pitch : 2 * a.out_pitch;
            if constexpr (DIRECT && DIR == 0 && CPT == 4 && WL_REALIGN_STORES &&
                          (P::kHalo == 1 || (WL_REALIGN97 && P::kReach == 1)) &&
                          !std::is_same_v<P, P_cdf53_polyphase_fwd> &&
                          !std::is_same_v<P, P_cdf97_polyphase_fwd>) {
                // Planes of any pitch / width: per plane row, the misalignment m
                // of the lane's first cell is warp-uniform (lanes are 4 cells
                // apart), so every lane stores the 16-byte block that starts
                // (4 - m) & 3 cells into its own cells, completed by the next
                // lane's first cells (shuffle) -- coalesced float4 rows; blocks
                // that leave the stored columns fall back to masked scalars.
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    const int qr = warp * R + r;
                    const int gy = gy0 + r;
                    if (!(qr >= H && qr < H + a.TH && gy >= a.ylo && gy < a.yhi)) continue;
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        float* const rp = pk[k] + r * step;
                        const int m = static_cast<int>((reinterpret_cast<uintptr_t>(rp) >> 2) & 3);
                        const int off = (4 - m) & 3;
                        float w0, w1, w2, w3;
                        if (m == 0) {
                            w0 = v[r][0][k]; w1 = v[r][1][k]; w2 = v[r][2][k]; w3 = v[r][3][k];
                        } else if (m == 1) {
                            w0 = v[r][3][k];
                            w1 = __shfl_down_sync(0xffffffffu, v[r][0][k], 1);
                            w2 = __shfl_down_sync(0xffffffffu, v[r][1][k], 1);
                            w3 = __shfl_down_sync(0xffffffffu, v[r][2][k], 1);
                        } else if (m == 2) {
                            w0 = v[r][2][k]; w1 = v[r][3][k];
                            w2 = __shfl_down_sync(0xffffffffu, v[r][0][k], 1);
                            w3 = __shfl_down_sync(0xffffffffu, v[r][1][k], 1);
                        } else {
                            w0 = v[r][1][k]; w1 = v[r][2][k]; w2 = v[r][3][k];
                            w3 = __shfl_down_sync(0xffffffffu, v[r][0][k], 1);
                        }
                        const int cl = CPT * lane + off;  // first cell of the block
                        const int gc = gx + off;          // its image cell column
                        if (cl >= HX && cl + 3 < HX + a.TW && gc >= 0 && gc + 3 < a.qw) {
                            *reinterpret_cast<float4*>(rp + off) = make_float4(w0, w1, w2, w3);
                        } else {
                            const float wv[4] = {w0, w1, w2, w3};
#pragma unroll
                            for (int t = 0; t < 4; ++t)
                                if (cl + t >= HX && cl + t < HX + a.TW && gc + t >= 0 && gc + t < a.qw)
                                    rp[off + t] = wv[t];
                        }
                    }
                }
            } else if constexpr (DIRECT && DIR == 1 && CPT == 2 && WL_INV_PAIR_STORES &&
                                 !std::is_same_v<P, P_cdf53_polyphase_inv> &&
                                 !std::is_same_v<P, P_cdf53_polyphase_star_inv>) {
                // Inverse image rows of any width: the lane's two cells are 4
                // consecutive pixels per row. Even pitch and base: float2 pairs,
                // or one float4 where the row's address is 16-byte aligned
                // (warp-uniform per row: lanes are 4 pixels apart); otherwise
                // element-wise. Per-cell column masks as below.
                const bool al8 = ((reinterpret_cast<uintptr_t>(a.out[0]) & 7) == 0) &&
                                 (a.out_pitch & 1) == 0 && (a.out_bstride[0] & 1) == 0;
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    const int qr = warp * R + r;
                    const int gy = gy0 + r;
                    if (!(qr >= H && qr < H + a.TH && gy >= a.ylo && gy < a.yhi)) continue;
                    const int cl = CPT * lane;
                    const bool ok0 = cl >= HX && cl < HX + a.TW && gx >= 0 && gx < a.qw;
                    const bool ok1 = cl + 1 >= HX && cl + 1 < HX + a.TW && gx + 1 >= 0 && gx + 1 < a.qw;
                    float* const p0 = pk[0] + r * step;
#pragma unroll
                    for (int h = 0; h < 2; ++h) {  // pixel rows 2y (LL HL) and 2y+1 (LH HH)
                        float* const p = p0 + h * a.out_pitch;
                        const float x0 = v[r][0][2 * h], x1 = v[r][0][2 * h + 1];
                        const float x2 = v[r][1][2 * h], x3 = v[r][1][2 * h + 1];
                        if (al8 && ok0 && ok1 && (reinterpret_cast<uintptr_t>(p) & 15) == 0) {
                            *reinterpret_cast<float4*>(p) = make_float4(x0, x1, x2, x3);
                        } else if (al8) {
                            if (ok0) *reinterpret_cast<float2*>(p) = make_float2(x0, x1);
                            if (ok1) *reinterpret_cast<float2*>(p + 2) = make_float2(x2, x3);
                        } else {
                            if (ok0) { p[0] = x0; p[1] = x1; }
                            if (ok1) { p[2] = x2; p[3] = x3; }
                        }
                    }
                }
            } else if constexpr (DIRECT && DIR == 1 && CPT == 4 && WL_INV_PAIR_STORES) {
                // Same for the CPT = 4 inverses (cdf97 Polyphase): 8 consecutive
                // pixels per lane and row -- two float4, or float2 + float4 +
                // float2 when the row is 8- but not 16-byte aligned.
                const bool al8 = ((reinterpret_cast<uintptr_t>(a.out[0]) & 7) == 0) &&
                                 (a.out_pitch & 1) == 0 && (a.out_bstride[0] & 1) == 0;
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    const int qr = warp * R + r;
                    const int gy = gy0 + r;
                    if (!(qr >= H && qr < H + a.TH && gy >= a.ylo && gy < a.yhi)) continue;
                    bool okc[4];
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const int cl = CPT * lane + j;
                        okc[j] = cl >= HX && cl < HX + a.TW && gx + j >= 0 && gx + j < a.qw;
                    }
                    const bool all = okc[0] && okc[1] && okc[2] && okc[3];
                    float* const p0 = pk[0] + r * step;
#pragma unroll
                    for (int h = 0; h < 2; ++h) {  // pixel rows 2y (LL HL) and 2y+1 (LH HH)
                        float* const p = p0 + h * a.out_pitch;
                        float x[8];
#pragma unroll
                        for (int j = 0; j < 4; ++j) {
                            x[2 * j] = v[r][j][2 * h];
                            x[2 * j + 1] = v[r][j][2 * h + 1];
                        }
                        if (al8 && all && (reinterpret_cast<uintptr_t>(p) & 15) == 0) {
                            *reinterpret_cast<float4*>(p) = make_float4(x[0], x[1], x[2], x[3]);
                            *reinterpret_cast<float4*>(p + 4) = make_float4(x[4], x[5], x[6], x[7]);
                        } else if (al8 && all) {
                            *reinterpret_cast<float2*>(p) = make_float2(x[0], x[1]);
                            *reinterpret_cast<float4*>(p + 2) = make_float4(x[2], x[3], x[4], x[5]);
                            *reinterpret_cast<float2*>(p + 6) = make_float2(x[6], x[7]);
                        } else {
#pragma unroll
                            for (int j = 0; j < 4; ++j) {
                                if (!okc[j]) continue;
                                if (al8) {
                                    *reinterpret_cast<float2*>(p + 2 * j) = make_float2(x[2 * j], x[2 * j + 1]);
                                } else {
                                    p[2 * j] = x[2 * j];
                                    p[2 * j + 1] = x[2 * j + 1];
                                }
                            }
                        }
                    }
                }
            } else if constexpr (DIRECT) {
                // element-wise stores under a per-cell column mask (any pitch,
                // any plane width); row validity is warp-uniform
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    const int qr = warp * R + r;
                    const int gy = gy0 + r;
                    const bool row_ok = qr >= H && qr < H + a.TH && gy >= a.ylo && gy < a.yhi;
#pragma unroll
                    for (int j = 0; j < CPT; ++j) {
                        const int cl = CPT * lane + j;  // cell column inside the compute region
                        const bool ok = row_ok && cl >= HX && cl < HX + a.TW && gx + j >= 0 &&
                                        gx + j < a.qw;
                        if (!ok) continue;
                        if (DIR == 0) {
#pragma unroll
                            for (int k = 0; k < 4; ++k) pk[k][r * step + j] = v[r][j][k];
                        } else {
                            float* p0 = pk[0] + r * step + 2 * j;
                            p0[0] = v[r][j][0];
                            p0[1] = v[r][j][1];
                            p0[a.out_pitch] = v[r][j][2];
                            p0[a.out_pitch + 1] = v[r][j][3];
                        }
                    }
                }
            } else if constexpr (CPT == 4) {
                // Whole-lane halo (lanes 0 and 31): a lane stores its 4 cells as
                // one aligned float4 per plane (qw = 0 mod 4, cx = 0 mod 4), or
                // nothing. Row validity is warp-uniform.
                const bool c_ok = lane >= HX / 4 && lane < 32 - HX / 4 && gx >= 0 && gx < a.qw;
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    const int qr = warp * R + r;
                    const int gy = gy0 + r;
#ifdef WL_DIAG_NO_STORE
                    const bool ok = a.ylo == -777;  // diagnostic: compute only (never true, not DCE-able)
#else
                    const bool ok = c_ok && qr >= H && qr < H + a.TH && gy >= a.ylo && gy < a.yhi;
#endif
                    if (DIR == 0) {
#pragma unroll
                        for (int k = 0; k < 4; ++k)
                            if (ok)
                                *reinterpret_cast<float4*>(pk[k] + r * step) =
                                    make_float4(v[r][0][k], v[r][1][k], v[r][2][k], v[r][3][k]);
                    } else {
                        float* p0 = pk[0] + r * step;
                        float* p1 = p0 + a.out_pitch;
                        if (ok) {
                            *reinterpret_cast<float4*>(p0) =
                                make_float4(v[r][0][0], v[r][0][1], v[r][1][0], v[r][1][1]);
                            *reinterpret_cast<float4*>(p0 + 4) =
                                make_float4(v[r][2][0], v[r][2][1], v[r][3][0], v[r][3][1]);
                            *reinterpret_cast<float4*>(p1) =
                                make_float4(v[r][0][2], v[r][0][3], v[r][1][2], v[r][1][3]);
                            *reinterpret_cast<float4*>(p1 + 4) =
                                make_float4(v[r][2][2], v[r][2][3], v[r][3][2], v[r][3][3]);
                        }
                    }
                }
            } else {
            // output columns of this tile, clipped to the image (partial tiles)
            const bool c0 = CPT * lane >= H && CPT * lane < H + a.TW && gx >= 0 && gx < a.qw;
            const bool c1 =
                CPT * lane + 1 >= H && CPT * lane + 1 < H + a.TW && gx + 1 >= 0 && gx + 1 < a.qw;
            // Branch-free, predicated stores: both cells (vector store) / only
            // the left / only the right cell. Row validity is warp-uniform.
            // With an even halo a lane's two cells are both stored or both halo
            // (only the "both" store exists); odd halos also need single cells.
            constexpr bool kPairs = WL_STORE_PAIRS && (H % 2 == 0);
            const bool both = c0 && c1, only0 = !kPairs && c0 && !c1, only1 = !kPairs && c1 && !c0;
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const int qr = warp * R + r;
                const int gy = gy0 + r;
                const bool row_ok = qr >= H && qr < H + a.TH && gy >= a.ylo && gy < a.yhi;
                if (DIR == 0) {
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        float* p = pk[k] + r * step;
                        if (row_ok && both)
                            *reinterpret_cast<float2*>(p) = make_float2(v[r][0][k], v[r][1][k]);
                        if (row_ok && only0) p[0] = v[r][0][k];
                        if (row_ok && only1) p[1] = v[r][1][k];
                    }
                } else {
                    float* p0 = pk[0] + r * step;
                    float* p1 = p0 + a.out_pitch;
                    if (row_ok && both) {
                        *reinterpret_cast<float4*>(p0) =
                            make_float4(v[r][0][0], v[r][0][1], v[r][1][0], v[r][1][1]);
                        *reinterpret_cast<float4*>(p1) =
                            make_float4(v[r][0][2], v[r][0][3], v[r][1][2], v[r][1][3]);
                    }
                    if (row_ok && only0) {
                        *reinterpret_cast<float2*>(p0) = make_float2(v[r][0][0], v[r][0][1]);
                        *reinterpret_cast<float2*>(p1) = make_float2(v[r][0][2], v[r][0][3]);
                    }
                    if (row_ok && only1) {
                        *reinterpret_cast<float2*>(p0 + 2) = make_float2(v[r][1][0], v[r][1][1]);
                        *reinterpret_cast<float2*>(p1 + 2) = make_float2(v[r][1][2], v[r][1][3]);
                    }
                }
            }
            }  // CPT == 2
        };
        body(std::integral_constant<int, 0>{});
    }
#ifdef WL_DIAG_TIMES
    if (dg && threadIdx.x == 0) {
        dg[2] = gtime();
        dg[3] = diag_tiles;
    }
#endif
}

// ------------------------------------------------------------------ host side
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiledFn encode_fn();
// Claim-counter slot for a launch on `stream` (wl_fast.cu); nullptr = static.
unsigned* sched_slot(cudaStream_t stream);
// Dynamic claims for (wavelet, direction)? (wl_fast.cu: default table,
// WL_DYN_MASK bit 2 * wavelet + direction overrides, WL_DYN=0 all off)
bool dyn_claims(int wavelet, int dir);

// 3-D map (w, h, nb images at `bstride` elements apart) of a float32 buffer;
// box = box_w x box_h x 1.
bool make_map(CUtensorMap* m, const float* base, int w, int h, long pitch, int nb, long bstride,
              int box_w, int box_h);

// Launch configuration per wavelet: (R, NW).
template <int WAVELET, int DIR>
struct Config;
// Tile geometry per wavelet, tuned on B200 at 16384^2 (fwd+inv pairs, see
// profiles/tuning_r01.md): cdf53 R=3 x NW=8 (3 CTAs/SM, 27 warps),
// cdf97 R=8 x NW=4 (deeper register rows, fewer exchanges per row).
// Geometry per (wavelet, direction): R rows per warp, NW compute warps, CPT
// cells per lane. Tuned on B200 at 16384^2 (profiles/tuning_r01*.txt):
// forwards use CPT = 4 (aligned float4 plane stores, sector-aligned tile
// boundaries), inverses CPT = 2 (their interleaved float4 image rows are
// already wide).
#ifndef WL_CPT_FWD
#define WL_CPT_FWD 4
#endif
#ifndef WL_CPT_INV
#define WL_CPT_INV 2
#endif
// exchange mode (1 = full) and CTAs-per-SM cap (0 = none) per configuration
#ifndef WL_XF53F
#define WL_XF53F 0
#endif
#ifndef WL_XF53I
#define WL_XF53I 0
#endif
#ifndef WL_XF97F
#define WL_XF97F 0
#endif
#ifndef WL_XF97I
#define WL_XF97I 0
#endif
#ifndef WL_MAXB53I
#define WL_MAXB53I 0
#endif
#ifndef WL_MAXB97I
#define WL_MAXB97I 2
#endif
// cdf53 forwards: 4 x 8 warps, 2-stage ring since the dynamic tile claims
// (3 x 8 with 3 stages before; 8192^2 -2..-5%, configs[4] 0.89 -> 0.94 of the
// copy peak, profiles/tuning_r02_s2.txt); Polyphase(*) keep 3 x 8 x 3 stages.
#ifndef WL_NS53F
#define WL_NS53F 2
#endif
#ifndef WL_NS53I
#define WL_NS53I 2
#endif
#ifndef WL_NS97F
#define WL_NS97F 2
#endif
#ifndef WL_NS97I
#define WL_NS97I 2
#endif
#ifndef WL_R53F
#define WL_R53F 4
#endif
#ifndef WL_NW53F
#define WL_NW53F 8
#endif
#ifndef WL_R97F
#define WL_R97F 5
#endif
#ifndef WL_NW97F
#define WL_NW97F 8
#endif
// cdf53 inverses: 4 x 8 (round 2, dynamic claims): 8192^2 -2..-8% over 3 x 8
#ifndef WL_R53I
#define WL_R53I 4
#endif
#ifndef WL_NW53I
#define WL_NW53I 8
#endif
// cdf97 inverses: 5 x 8 (40-row tiles, 16 compute warps per SM) since the
// dynamic tile claims; was 8 x 4 (profiles/tuning_r02_s2.txt: sweldens 8192^2
// 0.101 -> 0.094 ms, 16384^2 0.384 -> 0.331 ms)
#ifndef WL_R97I
#define WL_R97I 5
#endif
#ifndef WL_NW97I
#define WL_NW97I 8
#endif
template <>
struct Config<0, 0> {  // cdf53 forward, halo 1
    static constexpr int KR = 1;
    static constexpr int R = WL_R53F, NW = WL_NW53F, CPT = WL_CPT_FWD, NS = WL_NS53F;
    static constexpr bool XF = WL_XF53F;
    static constexpr int MAXB = 0;
};
template <>
struct Config<0, 1> {  // cdf53 inverse
    static constexpr int KR = 1;
    static constexpr int R = WL_R53I, NW = WL_NW53I, CPT = WL_CPT_INV, NS = WL_NS53I;
    static constexpr bool XF = WL_XF53I;
    static constexpr int MAXB = WL_MAXB53I;
};
template <>
struct Config<1, 0> {  // cdf97 forward, halo 2
    static constexpr int KR = 1;
    static constexpr int R = WL_R97F, NW = WL_NW97F, CPT = WL_CPT_FWD, NS = WL_NS97F;
    static constexpr bool XF = WL_XF97F;
    static constexpr int MAXB = 0;
};
template <>
struct Config<1, 1> {  // cdf97 inverse
    static constexpr int KR = 1;
    static constexpr int R = WL_R97I, NW = WL_NW97I, CPT = WL_CPT_INV, NS = WL_NS97I;
    static constexpr bool XF = WL_XF97I;
    static constexpr int MAXB = WL_MAXB97I;
};

// dd137 (reach 2: two ghost rows / lane-neighbour cells per side, halo 3),
// lifting schemes only (Polyphase(*) stays on the interpreter). Forward:
// CPT = 4, 32-row tiles (4 x 8 warps; the two-row edge exchange of 8 warps
// and the 36-row stage pair fit one CTA per SM).
#ifndef WL_R137
#define WL_R137 4
#endif
#ifndef WL_NW137
#define WL_NW137 8
#endif
// inverse: CPT = 2, 6 x 6 (3-18% faster than the forwards' geometry,
// profiles/tuning_r02_s2.txt)
#ifndef WL_R137I
#define WL_R137I 6
#endif
#ifndef WL_NW137I
#define WL_NW137I 6
#endif
#ifndef WL_CPT137I
#define WL_CPT137I 2
#endif
#ifndef WL_CPT137F
#define WL_CPT137F 4
#endif
template <>
struct Config<2, 0> {
    static constexpr int R = WL_R137, NW = WL_NW137, CPT = WL_CPT137F, NS = 2;
    static constexpr bool XF = false;
    static constexpr int MAXB = 0;
    static constexpr int KR = 2;
};
template <>
struct Config<2, 1> {
    static constexpr int R = WL_R137I, NW = WL_NW137I, CPT = WL_CPT137I, NS = 2;
    static constexpr bool XF = false;
    static constexpr int MAXB = 0;
    static constexpr int KR = 2;
};

// Per-scheme override of the geometry (scheme = SchemeKind index). The cdf97
// Polyphase inverse (one 126-MAC neighbour epoch: FP32-issue heavy) runs 26-30%
// faster with the forwards' CPT = 4 layout; Polyphase* and cdf53 do not gain
// (profiles/tuning_r01_poly_inv.txt).
#ifndef WL_POLY_INV_CPT4
#define WL_POLY_INV_CPT4 1
#endif
template <int WAVELET, int DIR, int SCHEME>
struct SchemeConfig : Config<WAVELET, DIR> {};
// Geometry of the direct-load instantiation of a program (see WL_DIRECT_R).
template <int WAVELET, int DIR, int SCHEME, class C = SchemeConfig<WAVELET, DIR, SCHEME>>
struct DirectConfigOf : C {  // forwards only (inverses keep the TMA geometry); WL_DIRECT_R=0 off
    static constexpr bool kOwn = DIR == 0 && WL_DIRECT_R > 0;
    // cdf97 Polyphase forward: 4-row warps (its 126-MAC epoch is 14% slower on 3)
    static constexpr int kR = WAVELET == 1 && SCHEME == 7 && WL_DIRECT_R == 3 ? 4 : WL_DIRECT_R;
    static constexpr int R = !kOwn ? C::R : (kR > 2 * C::KR ? kR : 2 * C::KR);
    static constexpr int NW = !kOwn || C::NW < WL_DIRECT_NW ? C::NW : WL_DIRECT_NW;  // 2 x 288 threads: <= 113 regs
};
#if WL_POLY_INV_CPT4
#ifndef WL_POLY_R
#define WL_POLY_R 3
#endif
#ifndef WL_POLY_NS_FWD
#define WL_POLY_NS_FWD 2
#endif
#ifndef WL_POLY_NS_INV
#define WL_POLY_NS_INV 2
#endif
#ifndef WL_POLY_NW
#define WL_POLY_NW 10
#endif
template <int SCHEME>
struct PolyInv {
    static constexpr int KR = 1;
    static constexpr int R = WL_POLY_R, NW = WL_POLY_NW, CPT = 4, NS = WL_POLY_NS_INV;
    static constexpr bool XF = false;
    static constexpr int MAXB = 0;
};
template <>
struct SchemeConfig<1, 1, 7> : PolyInv<7> {};  // cdf97 polyphase inverse
#endif
// cdf97 Polyphase forward: 6 exchanged component rows (its single neighbour
// epoch reads 4 components above, 2 below): 32-row tiles and a 2-stage ring
// (profiles/tuning_r01_tiles97.txt).
template <>
struct SchemeConfig<1, 0, 7> : Config<1, 0> {
    static constexpr int NS = WL_POLY_NS_FWD;
    static constexpr int R = WL_POLY_R;  // 30-row tiles x 10 warps (profiles/tuning_r01_poly.txt)
    static constexpr int NW = WL_POLY_NW;
};

// cdf97 Iwahashi(*) / Explosive(*) forwards (three neighbour epochs): 40-row
// tiles as 4 x 10 warps, 2-4% faster than 5 x 8 (profiles/tuning_r02_s2.txt,
// variant f410); Sweldens and Monolithic(*) keep 5 x 8.
#ifndef WL_R97F_IE
#define WL_R97F_IE 4
#endif
#ifndef WL_NW97F_IE
#define WL_NW97F_IE 10
#endif
template <int SCHEME>
struct Fwd97IE : Config<1, 0> {
    static constexpr int R = WL_R97F_IE, NW = WL_NW97F_IE;
};
template <>
struct SchemeConfig<1, 0, 1> : Fwd97IE<1> {};
template <>
struct SchemeConfig<1, 0, 2> : Fwd97IE<2> {};
template <>
struct SchemeConfig<1, 0, 3> : Fwd97IE<3> {};
template <>
struct SchemeConfig<1, 0, 4> : Fwd97IE<4> {};
// cdf97 Polyphase* forward (one 4x4 matrix epoch of reach 1 after the local
// steps): A/B knobs, default = the generic cdf97 forward geometry.
#ifndef WL_R97F_PS
#define WL_R97F_PS WL_R97F
#endif
#ifndef WL_NW97F_PS
#define WL_NW97F_PS WL_NW97F
#endif
template <>
struct SchemeConfig<1, 0, 8> : Config<1, 0> {
    static constexpr int R = WL_R97F_PS, NW = WL_NW97F_PS;
};

template <int SCHEME>
struct Fwd53Poly : Config<0, 0> {
    static constexpr int R = 3, NS = 3;
};
template <>
struct SchemeConfig<0, 0, 7> : Fwd53Poly<7> {};
template <>
struct SchemeConfig<0, 0, 8> : Fwd53Poly<8> {};

// Tuning knob: one extra per-scheme override from the compiler command line
// (-DWL_OVR_W=w -DWL_OVR_D=d -DWL_OVR_S=s -DWL_OVR_R=.. -DWL_OVR_NW=.. -DWL_OVR_NS=..
// -DWL_OVR_XF=..), for A/B builds.
#ifdef WL_OVR_S
template <>
struct SchemeConfig<WL_OVR_W, WL_OVR_D, WL_OVR_S> : Config<WL_OVR_W, WL_OVR_D> {
    static constexpr int R = WL_OVR_R, NW = WL_OVR_NW, NS = WL_OVR_NS;
    static constexpr bool XF = WL_OVR_XF;
};
#endif

// cdf97 Monolithic / Monolithic* inverses: the full exchange measured faster
// at 8 x 4 (profiles/tuning_r01_exchange.txt); at 5 x 8 the minimal exchange
// keeps two CTAs per SM and wins (0.103 / 0.096 ms vs 0.111 / 0.106 ms at
// 8192^2, profiles/tuning_r02_s2.txt). Knobs for A/B builds.
#ifndef WL_RMONO97I
#define WL_RMONO97I WL_R97I
#endif
#ifndef WL_XFMONO97I
#define WL_XFMONO97I WL_XF97I
#endif
template <>
struct SchemeConfig<1, 1, 5> : Config<1, 1> {
    static constexpr bool XF = WL_XFMONO97I;
    static constexpr int R = WL_RMONO97I;
};
template <>
struct SchemeConfig<1, 1, 6> : Config<1, 1> {
    static constexpr bool XF = WL_XFMONO97I;
    static constexpr int R = WL_RMONO97I;
};

struct Plan {
    FastArgs args;
    int tiles_y;
    bool ok;
};

// Tile grid of the fast path.
//  * periodic: the grid covers the whole image (one extra tile row/column on
//    the top/left, t0 = -1); border tiles load wrapped cells (exact).
//  * symmetric: only tiles whose compute region lies inside the image; the
//    frame around them is the interpreter's (per-step mirroring).
//  * strip window (L.yhi > 0, periodic only): tile rows cover the stored rows
//    [ylo, yhi) only; the rows around them are halo rows physically present
//    in the buffer (ylo >= H + 1 and yhi <= qh - H - 1 keep every stored
//    cell's dependency cone and the tiles' ghost rows inside the buffer).
//  * periodic plans (whole image or strip window; `legacy` = the former grid,
//    an A/B knob): tile (0, 0) stores cell (0, 0) onwards -- only its
//    reach + 1 ghost rows / halo columns wrap -- and the last tile row /
//    column is clamped to end at the image edge (overlapping its neighbour,
//    which writes the same values), so no tile computes wrapped cells it does
//    not store: the former plan (first row/column of tiles BEFORE the image,
//    last ones past its end) cost 7-10% redundant work at 8192^2 and its
//    nearly-all-wrapped edge tiles made the launch's tail.
inline Plan plan_tiles(const WlLevel& L, int H, int R, int NW, int CPT, bool no_mirror = false,
                       bool legacy = false, int KR = 1) {
    Plan p{};
    p.args.xlast = p.args.ylast = 0x7fffffff;
    const int nb = L.nb > 1 ? L.nb : 1;
    p.args.ylo = 0;
    p.args.yhi = L.qh;
    const int TWC = 32 * CPT;
    // TMA requires the innermost box start to be 16-byte aligned: the inverse
    // boxes start at cell column X0 - HX + tx*TW of a float32 plane, so TW is
    // rounded down to a multiple of 4 there (the forward starts at pixel
    // column 2*(...) and 2*(64 - 2H) is a multiple of 4 for H = 1, 2).
    // CPT = 4: HX = 4, TW = 120; tile column 0 starts its compute region at
    // cell -4 (X0 = 0) so every tile's stored columns start at 120*tx.
    const int HX = CPT == 4 ? 4 : H;
    const int TW = CPT == 4 ? TWC - 2 * HX
                            : (L.direction == 0 ? TWC - 2 * H : ((TWC - 2 * H) & ~3));
    const int TH = NW * R - 2 * H;
    const bool wide = CPT == 4;
    // Symmetric images whose width is a multiple of the lane width run the
    // whole-image grid too: border tiles mirror their ghost cells per step
    // (kernel `mtile`); otherwise only interior tiles run here and the frame
    // goes to the interpreter.
    // A symmetric WINDOW (strip of a symmetric row-strip pyramid) is planned
    // as the whole buffer [0, qh): the buffer edges are either the image's own
    // (mirrored, exact) or at least H + 1 halo rows away from every stored row
    // (their wrong mirroring never reaches a stored cell); the stores keep to
    // [ylo, yhi).
    const bool sym_window = L.boundary == 1 && L.yhi > 0;
    bool full_sym = L.boundary == 1 && L.qw >= 2 && L.qh >= 2 &&
                    L.qw % CPT == 0 && WL_SYM_FAST && !no_mirror && KR == 1;
    // Row offset of the symmetric grid: every tile whose compute rows hold
    // image row 0 must not have it as a warp's last row (its mirror source,
    // row 1, would sit in the next warp), nor row qh-1 as a warp's first row.
    const int THs = NW * R - 2 * H;
    auto rows_ok = [&](int y0) {
        for (int ty = -1;; ++ty) {
            const int c0 = y0 + ty * THs - H, c1 = c0 + NW * R;  // compute rows [c0, c1)
            if (c0 > L.qh) return true;
            if (c0 <= 0 && 0 < c1 && (0 - c0) % R == R - 1) return false;
            if (c0 <= L.qh - 1 && L.qh - 1 < c1 && (L.qh - 1 - c0) % R == 0) return false;
        }
    };
    int ysym = 0;
    if (full_sym) {
        for (int y0 = H + 1; y0 <= THs && !ysym; ++y0)
            if (rows_ok(y0)) ysym = y0;
        full_sym = ysym > 0;
    }
    const bool whole = L.boundary == 0 || (L.yhi > 0 && !sym_window) || full_sym;
    int X0 = wide ? (whole ? 0 : HX) : H;
    const int Y0 = full_sym ? ysym : H + KR;
    const int tx0 = wide ? 0 : -1;  // periodic plans
    int tx, ty;
    int y0 = Y0;
    p.args.mirror = full_sym ? 1 : 0;
    if (sym_window && (L.ylo < 0 || L.yhi > L.qh || L.yhi <= L.ylo)) return p;  // ok = false
    if (L.yhi > 0 && !sym_window) {
        if (L.boundary != 0 || L.ylo < H + KR || L.yhi > L.qh - H - KR || L.yhi <= L.ylo)
            return p;  // ok = false
        tx = (L.qw - X0 > 0 ? (L.qw - X0 + TW - 1) / TW : 0) - tx0;
        ty = (L.yhi - L.ylo + TH - 1) / TH;
        y0 = L.ylo;
        p.args.tx0 = tx0;
        p.args.ty0 = 0;
        p.args.wrap = 1;
        p.args.ylo = L.ylo;
        p.args.yhi = L.yhi;
    } else if (whole) {
        tx = (L.qw - X0 > 0 ? (L.qw - X0 + TW - 1) / TW : 0) - tx0;
        ty = (L.qh - Y0 > 0 ? (L.qh - Y0 + TH - 1) / TH : 0) + 1;
        p.args.tx0 = tx0;
        p.args.ty0 = -1;
        p.args.wrap = full_sym ? 0 : 1;
    } else {
        const int c0 = X0 - HX;  // first compute column of tile 0 (>= 0)
        tx = L.qw - c0 >= TWC ? (L.qw - c0 - TWC) / TW + 1 : 0;
        const int span = L.qh - (Y0 - H - KR);  // rows available from the first ghost row
        ty = span >= NW * R + 2 * KR ? (span - (NW * R + 2 * KR)) / TH + 1 : 0;
        p.args.tx0 = p.args.ty0 = 0;
        p.args.wrap = 0;
    }
    if (WL_PLAN_V2 && L.boundary == 0 && !legacy && (whole || (L.yhi > 0 && !sym_window))) {
        // X0 - HX = -4: box starts stay 16-byte aligned (TW = 0 mod 4 when CPT = 2)
        const int Xp = wide ? 0 : H - 4;
        tx = L.qw - Xp > 0 ? (L.qw - Xp + TW - 1) / TW : 0;
        const int xr = L.qw - TW - Xp;  // last origin rounded UP to the 4-cell grid
        p.args.xlast = Xp + (xr > 0 ? (xr + 3) / 4 * 4 : 0);
        p.args.tx0 = 0;
        X0 = Xp;
        if (whole) {
            ty = (L.qh + TH - 1) / TH;
            y0 = 0;
            p.args.ylast = L.qh - TH > 0 ? L.qh - TH : 0;
            p.args.ty0 = 0;
        } else {
            p.args.ylast = L.yhi - TH > L.ylo ? L.yhi - TH : L.ylo;
        }
    }
    p.args.tiles_x = tx;
    p.tiles_y = ty;
    p.args.ntiles_img = tx * ty;
    p.args.ntiles = nb * tx * ty;
    p.args.X0 = X0;
    p.args.Y0 = y0;
    p.args.TW = TW;
    p.args.TH = TH;
    p.args.qw = L.qw;
    p.args.qh = L.qh;
    if (sym_window) {
        p.args.ylo = L.ylo;
        p.args.yhi = L.yhi;
    }
    p.ok = tx > 0 && ty > 0 && (long)nb * tx * ty < (1l << 31);
    return p;
}

// Kernel arguments and tensor maps of one level.
template <class P, int DIR, int R, int NW, int CPT, int NS, bool XF>
bool level_args(const WlLevel& L, const Plan& plan, FastArgs& a, CUtensorMap (&maps)[4]) {
    using G = Geometry<R, NW, CPT, NS, xch_comps<P, XF>(), P::kReach>;
    constexpr int TWC = G::TWC;
    a = plan.args;
    const int nb = L.nb > 1 ? L.nb : 1;
    for (int k = 0; k < 4; ++k) {
        a.in_bstride[k] = nb > 1 ? L.in_bstride[k] : 0;
        a.out_bstride[k] = nb > 1 ? L.out_bstride[k] : 0;
    }
    if (DIR == 0) {
        static_assert((2 * G::kRows) % WL_FWD_SPLIT == 0, "split must divide the tile rows");
        if (!make_map(&maps[0], L.in[0], 2 * L.qw, 2 * L.qh, L.in_pitch, nb, a.in_bstride[0],
                      2 * TWC, 2 * G::kRows / WL_FWD_SPLIT))
            return false;
        maps[1] = maps[2] = maps[3] = maps[0];
        for (int k = 0; k < 4; ++k) a.out[k] = L.out[k];
    } else {
        for (int k = 0; k < 4; ++k)
            if (!make_map(&maps[k], L.in[k], L.qw, L.qh, L.in_pitch, nb, a.in_bstride[k], TWC,
                          G::kRows))
                return false;
        a.out[0] = L.out[0];
        a.out[1] = a.out[2] = a.out[3] = nullptr;
    }
    for (int k = 0; k < 4; ++k) a.in[k] = L.in[k];
    a.xflag_a = L.xflag_a;
    a.xflag_b = L.xflag_b;
    a.xepoch = L.xepoch;
    a.xerr = L.xerr;
    a.diag = wl_diag_ptr();
    a.in_pitch = L.in_pitch;
    a.out_pitch = L.out_pitch;
    a.scaling = L.scaling && wl_host_program(L.prog).has_scale;
    a.scale = wl_host_program(L.prog).scale;
    return true;
}

// Persistent grid size of a kernel variant: SMs x resident CTAs (cached per device).
template <int R, int NW, int CPT, int NS, int NXC, int MAXB, int KR, class Kern>
int grid_cap(Kern kern, int* cache) {
    using G = Geometry<R, NW, CPT, NS, NXC, KR>;
    int dev = 0;
    cudaGetDevice(&dev);
    int& mb = cache[dev & 63];
    if (mb != 0) return mb;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)G::kSmemBytes);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, (NW + 1) * 32, G::kSmemBytes);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (MAXB > 0 && per_sm > MAXB) per_sm = MAXB;
    mb = (per_sm > 0 ? per_sm : 1) * sms;
    if (getenv("WL_VERBOSE"))
        fprintf(stderr, "[wl] fast_kernel R=%d NW=%d CPT=%d NS=%d smem=%zu B: %d CTA/SM\n", R, NW,
                CPT, NS, (size_t)G::kSmemBytes, per_sm);
    return mb;
}

template <class P, int DIR, int R, int NW, int CPT, int NS, bool XF, int MAXB>
cudaError_t launch(const WlLevel& L, const Plan& plan, cudaStream_t stream) {
    constexpr int NXC = xch_comps<P, XF>();
    using G = Geometry<R, NW, CPT, NS, NXC, P::kReach>;
    CUtensorMap maps[4];
    KArgs k{};
    if (!level_args<P, DIR, R, NW, CPT, NS, XF>(L, plan, k.lv[0], maps))
        return cudaErrorInvalidValue;
    static int cap_norm[64] = {}, cap_mirr[64] = {};
    auto run = [&](auto kern, int* cache, int filter) -> cudaError_t {
        const int mb = grid_cap<R, NW, CPT, NS, NXC, MAXB, P::kReach>(kern, cache);
        KArgs f = k;
        f.lv[0].filter = filter;
        f.lv[0].sched = f.lv[0].ntiles > mb && dyn_claims(L.wavelet, DIR) ? sched_slot(stream) : nullptr;
        const int grid = f.lv[0].ntiles < mb ? f.lv[0].ntiles : mb;
        cudaError_t le = launch_pdl(kern, dim3(grid), dim3((NW + 1) * 32), G::kSmemBytes,
                                    stream, maps[0], maps[1], maps[2], maps[3], f);
        wl_count_launch();
        return le != cudaSuccess ? le : cudaGetLastError();
    };
    if constexpr (P::kReach > 1) {  // no mirrored variant (plans never set mirror)
        (void)cap_mirr;
        if (k.lv[0].mirror) return cudaErrorNotSupported;
        return run(fast_kernel<P, DIR, R, NW, CPT, NS, XF, false>, cap_norm, 0);
    } else {
        if (!k.lv[0].mirror) return run(fast_kernel<P, DIR, R, NW, CPT, NS, XF, false>, cap_norm, 0);
        // symmetric whole-image plan: interior tiles on the plain kernel, the ring
        // of border tiles on the mirroring variant (same grid, disjoint tiles)
        cudaError_t e = run(fast_kernel<P, DIR, R, NW, CPT, NS, XF, false>, cap_norm, 1);
        if (e != cudaSuccess) return e;
        return run(fast_kernel<P, DIR, R, NW, CPT, NS, XF, true>, cap_mirr, 2);
    }
}

// Direct-load launch (no TMA, element-wise stores): shapes the TMA path
// cannot take. Plain plans only (periodic whole image, strip windows, or the
// symmetric interior grid + interpreter frame).
template <class P, int DIR, int R, int NW, int CPT, int NS, bool XF, int MAXB>
cudaError_t launch_direct(const WlLevel& L, const Plan& plan, cudaStream_t stream) {
    constexpr int NXC = xch_comps<P, XF>();
    using G = Geometry<R, NW, CPT, NS, NXC, P::kReach>;
    if (plan.args.mirror) return cudaErrorNotSupported;
    KArgs k{};
    FastArgs& a = k.lv[0];
    a = plan.args;
    const int nb = L.nb > 1 ? L.nb : 1;
    for (int q = 0; q < 4; ++q) {
        a.in[q] = L.in[q];
        a.out[q] = DIR == 0 ? L.out[q] : (q == 0 ? L.out[0] : nullptr);
        a.in_bstride[q] = nb > 1 ? L.in_bstride[q] : 0;
        a.out_bstride[q] = nb > 1 ? L.out_bstride[q] : 0;
    }
    a.xflag_a = a.xflag_b = nullptr;
    a.sched = nullptr;  // no producer warp: static tiles
    a.diag = wl_diag_ptr();
    a.in_pitch = L.in_pitch;
    a.out_pitch = L.out_pitch;
    a.scaling = L.scaling && wl_host_program(L.prog).has_scale;
    a.scale = wl_host_program(L.prog).scale;
    a.filter = 0;
    constexpr size_t smem = (size_t)G::kXchFloats * 4 + 16 * NS;
    auto kern = fast_kernel<P, DIR, R, NW, CPT, NS, XF, false, true>;
    static int cap[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    int& mb = cap[dev & 63];
    if (mb == 0) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        int per_sm = 0, sms = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, (NW + 1) * 32, smem);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        mb = (per_sm > 0 ? per_sm : 1) * sms;
    }
    const int grid = a.ntiles < mb ? a.ntiles : mb;
    CUtensorMap none{};
    cudaError_t le = launch_pdl(kern, dim3(grid), dim3((NW + 1) * 32), smem, stream, none, none,
                                none, none, k);
    wl_count_launch();
    return le != cudaSuccess ? le : cudaGetLastError();
}

}  // namespace wlfast
