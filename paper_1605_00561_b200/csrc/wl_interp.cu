// Generic tile interpreter for every (wavelet, scheme, direction, boundary).
//
// One CTA owns a TQ x TQ tile of component cells (quads) plus the program's
// halo. The step list of the program (gen/programs_gen.h) is evaluated from
// __constant__ tap tables, exactly in the reference's apply_step summation
// order (transform.cpp:100-125), with shared-memory ping-pong buffers:
//
//   * a neighbour-reading step publishes the current cell values to shared
//     memory and waits on ONE block barrier, so the number of __syncthreads()
//     per tile equals count_barriers (schemes.cpp:193-198) -- the first of
//     them is the data-availability barrier after the load;
//   * local (0,0) steps (the "star" scalar steps) run in registers on the
//     thread's own cells and need no barrier (each thread keeps its cells
//     for the whole program).
//
// Boundaries: periodic tiles load the wrapped neighbourhood (load-time wrap is
// exact for periodic, parsim.cpp:253-257); symmetric tiles re-resolve every
// out-of-image read on the component grid per step (transform.cpp:114-115),
// which reproduces the reference's per-step whole-point mirroring exactly.
//
// This engine is the correctness baseline and the path for symmetric border
// handling, dd137 and Convolution; the fast register engine (wl_fast.cu)
// takes the hot cdf53/cdf97 lifting programs.
#include <cuda_runtime.h>

#include "gen/programs_gen.h"
#include "wl_internal.h"

namespace {

constexpr int TQ = 32;        // output cells per tile side
constexpr int NT = 256;       // threads per CTA
constexpr int MAXH = 6;       // largest tile halo: 2 x dd137's reach (symmetric)
constexpr int RSMAX = TQ + 2 * MAXH;
constexpr int K = (RSMAX * RSMAX + NT - 1) / NT;  // cells per thread

__constant__ WlTap c_taps[WL_NUM_TAPS] = WL_TAPS_INIT;
__constant__ WlStep c_steps[WL_NUM_STEPS] = WL_STEPS_INIT;
__constant__ WlProgram c_progs[60] = WL_PROGRAMS_INIT;
__constant__ WlConvTap c_conv[WL_NUM_CONV_TAPS] = WL_CONV_TAPS_INIT;

// transform.cpp:59-72 resolve_index.
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

__device__ __forceinline__ float pick(const float (&v)[4], int i) {
    return i == 0 ? v[0] : i == 1 ? v[1] : i == 2 ? v[2] : v[3];
}

template <int DIR>
__global__ void __launch_bounds__(NT) interp_kernel(const WlLevel L, const WlRects RC) {
    extern __shared__ float sm[];
    const WlProgram& P = c_progs[L.prog];
    const bool sym = L.boundary == 1;
    // Symmetric: a read past the image border is mirrored back inwards, so
    // next to a border the up- and down-reach (left and right) add up.
    const int H = sym ? 2 * P.halo : P.halo;
    // Linear block index -> (rectangle, tile) of the output region; each
    // rectangle has its own tile shape (TY x TX output cells; thin frame
    // strips get flat tiles so little work is spent on discarded halo).
    int b = blockIdx.x, rect = 0;
    int tiles_x = (RC.nx[0] + RC.tx[0] - 1) / RC.tx[0];
    while (rect + 1 < RC.n && b >= tiles_x * ((RC.ny[rect] + RC.ty[rect] - 1) / RC.ty[rect])) {
        b -= tiles_x * ((RC.ny[rect] + RC.ty[rect] - 1) / RC.ty[rect]);
        ++rect;
        tiles_x = (RC.nx[rect] + RC.tx[rect] - 1) / RC.tx[rect];
    }
    const int TY = RC.ty[rect], TX = RC.tx[rect];
    const int RSY = TY + 2 * H, RS = TX + 2 * H;  // region rows, region row length
    const int plane = RSY * RS;
    const int ty = b / tiles_x, tx = b - (b / tiles_x) * tiles_x;
    const int ry0 = RC.y0[rect] + ty * TY, rx0 = RC.x0[rect] + tx * TX;  // tile output origin
    const int ry1 = min(ry0 + TY, RC.y0[rect] + RC.ny[rect]);
    const int rx1 = min(rx0 + TX, RC.x0[rect] + RC.nx[rect]);
    const int oy = ry0 - H, ox = rx0 - H;

    float v[K][4];
    int ly[K], lx[K];
    bool live[K];  // cell participates in the computation

#pragma unroll
    for (int k = 0; k < K; ++k) {
        const int idx = threadIdx.x + k * NT;
        ly[k] = idx / RS;
        lx[k] = idx - ly[k] * RS;
        const int gy = oy + ly[k], gx = ox + lx[k];
        live[k] = idx < plane && (!sym || (gy >= 0 && gy < L.qh && gx >= 0 && gx < L.qw));
        v[k][0] = v[k][1] = v[k][2] = v[k][3] = 0.f;
        if (!live[k]) continue;
        const int ry = resolve(gy, L.qh, L.boundary), rx = resolve(gx, L.qw, L.boundary);
        if (DIR == 0) {
            // polyphase_split (transform.cpp:74-86) fused into the load.
            const float* r0 = L.in[0] + (long)(2 * ry) * L.in_pitch + 2 * rx;
            v[k][0] = r0[0];
            v[k][1] = r0[1];
            v[k][2] = r0[L.in_pitch];
            v[k][3] = r0[L.in_pitch + 1];
        } else {
            const long o = (long)ry * L.in_pitch + rx;
#pragma unroll
            for (int c = 0; c < 4; ++c) v[k][c] = L.in[c][o];
            if (L.scaling && P.has_scale) {  // undo scaling first (transform.cpp:180)
                v[k][0] *= P.scale;
                v[k][3] /= P.scale;
            }
        }
    }

    int cur = 0;
    for (int si = 0; si < P.nsteps; ++si) {
        const WlStep st = c_steps[P.step0 + si];
        int t0[4];
        t0[0] = st.tap0;
        t0[1] = t0[0] + st.dst_n[0];
        t0[2] = t0[1] + st.dst_n[1];
        t0[3] = t0[2] + st.dst_n[2];
        if (st.reads_nbr) {
            float* b = sm + cur * 4 * plane;
#pragma unroll
            for (int k = 0; k < K; ++k)
                if (live[k])
#pragma unroll
                    for (int c = 0; c < 4; ++c) b[c * plane + ly[k] * RS + lx[k]] = v[k][c];
            __syncthreads();  // one barrier per neighbour-reading step
#pragma unroll
            for (int k = 0; k < K; ++k) {
                if (!live[k]) continue;
                float o[4];
#pragma unroll
                for (int d = 0; d < 4; ++d) {
                    float acc = 0.f;
                    for (int t = t0[d]; t < t0[d] + st.dst_n[d]; ++t) {
                        const WlTap tp = c_taps[t];
                        int yy = ly[k] + tp.dr, xx = lx[k] + tp.dc;
                        if (sym) {
                            const int gy = oy + yy, gx = ox + xx;
                            if (gy < 0 || gy >= L.qh) yy = resolve(gy, L.qh, 1) - oy;
                            if (gx < 0 || gx >= L.qw) xx = resolve(gx, L.qw, 1) - ox;
                        }
                        yy = min(max(yy, 0), RSY - 1);
                        xx = min(max(xx, 0), RS - 1);
                        acc = fmaf(tp.c, b[tp.src * plane + yy * RS + xx], acc);
                    }
                    o[d] = acc;
                }
#pragma unroll
                for (int d = 0; d < 4; ++d) v[k][d] = o[d];
            }
            cur ^= 1;
        } else {
#pragma unroll
            for (int k = 0; k < K; ++k) {
                if (!live[k]) continue;
                float o[4];
#pragma unroll
                for (int d = 0; d < 4; ++d) {
                    float acc = 0.f;
                    for (int t = t0[d]; t < t0[d] + st.dst_n[d]; ++t) {
                        const WlTap tp = c_taps[t];
                        acc = fmaf(tp.c, pick(v[k], tp.src), acc);
                    }
                    o[d] = acc;
                }
#pragma unroll
                for (int d = 0; d < 4; ++d) v[k][d] = o[d];
            }
        }
    }

#pragma unroll
    for (int k = 0; k < K; ++k) {
        const int gy = oy + ly[k], gx = ox + lx[k];
        if (!live[k] || gy < ry0 || gy >= ry1 || gx < rx0 || gx >= rx1 || gy >= L.qh ||
            gx >= L.qw)
            continue;
        if (DIR == 0) {
            if (L.scaling && P.has_scale) {  // scale_planes (transform.cpp:154-159)
                v[k][0] *= P.scale;
                v[k][3] /= P.scale;
            }
            const long o = (long)gy * L.out_pitch + gx;
#pragma unroll
            for (int c = 0; c < 4; ++c) L.out[c][o] = v[k][c];
        } else {
            // polyphase_merge (transform.cpp:88-98) fused into the store.
            float* r0 = L.out[0] + (long)(2 * gy) * L.out_pitch + 2 * gx;
            r0[0] = v[k][0];
            r0[1] = v[k][1];
            r0[L.out_pitch] = v[k][2];
            r0[L.out_pitch + 1] = v[k][3];
        }
    }
}

// Direct 2-D analysis filters at subsampled positions (transform.cpp:129-152),
// mirrored / wrapped on the IMAGE grid at load time (exact: a single pass).
constexpr int CR_MAX = 6;  // dd137 filter reach (13 taps)
constexpr int CS = 2 * TQ + 2 * CR_MAX;

__global__ void __launch_bounds__(NT) conv_kernel(const WlLevel L) {
    __shared__ float px[CS * CS];
    const WlProgram& P = c_progs[L.prog];
    const int R = P.creach;
    const int side = 2 * TQ + 2 * R;
    const int w = 2 * L.qw, h = 2 * L.qh;
    const int py0 = 2 * blockIdx.y * TQ - R, px0 = 2 * blockIdx.x * TQ - R;
    for (int i = threadIdx.x; i < side * side; i += NT) {
        const int y = i / side, x = i - (i / side) * side;
        const int ry = resolve(py0 + y, h, L.boundary), rx = resolve(px0 + x, w, L.boundary);
        px[y * side + x] = L.in[0][(long)ry * L.in_pitch + rx];
    }
    __syncthreads();  // the single data-availability barrier
    const int pr[4] = {0, 0, 1, 1}, pc[4] = {0, 1, 0, 1};
    for (int q = threadIdx.x; q < TQ * TQ; q += NT) {
        const int qy = q / TQ, qx = q - (q / TQ) * TQ;
        const int gy = blockIdx.y * TQ + qy, gx = blockIdx.x * TQ + qx;
        if (gy >= L.qh || gx >= L.qw) continue;
        float o[4];
        int t = P.conv0;
#pragma unroll
        for (int comp = 0; comp < 4; ++comp) {
            float acc = 0.f;
            const int by = 2 * qy + pr[comp] + R, bx = 2 * qx + pc[comp] + R;
            for (int e = 0; e < P.convn[comp]; ++e, ++t) {
                const WlConvTap tp = c_conv[t];
                acc = fmaf(tp.c, px[(by + tp.dr) * side + bx + tp.dc], acc);
            }
            o[comp] = acc;
        }
        if (L.scaling && P.has_scale) {
            o[0] *= P.scale;
            o[3] /= P.scale;
        }
        const long off = (long)gy * L.out_pitch + gx;
#pragma unroll
        for (int c = 0; c < 4; ++c) L.out[c][off] = o[c];
    }
}

const WlProgram h_progs[60] = WL_PROGRAMS_INIT;
const WlStep h_steps[WL_NUM_STEPS] = WL_STEPS_INIT;

}  // namespace

const WlProgram& wl_host_program(int prog) { return h_progs[prog]; }
const WlStep* wl_host_steps() { return h_steps; }

cudaError_t wl_launch_interp(const WlLevel& L, cudaStream_t stream) {
    WlRects R{};
    R.n = 1;
    R.ny[0] = L.qh;
    R.nx[0] = L.qw;
    R.ty[0] = R.tx[0] = TQ;
    return wl_launch_interp_rects(L, R, stream);
}

cudaError_t wl_launch_interp_rects(const WlLevel& L, const WlRects& RC, cudaStream_t stream) {
    const WlProgram& P = h_progs[L.prog];
    const int H = L.boundary == 1 ? 2 * P.halo : P.halo;
    const int cap = NT * K;  // region cells one CTA holds
    // Drop empty rectangles and pick a tile shape per rectangle: 32x32 in
    // general, flat tiles for thin strips (the frame around the fast engine).
    WlRects R{};
    long blocks = 0;
    size_t cells = 0;
    for (int i = 0; i < RC.n; ++i) {
        if (RC.ny[i] <= 0 || RC.nx[i] <= 0) continue;
        int ty = TQ, tx = TQ;
        if (RC.ny[i] < TQ && RC.ny[i] <= RC.nx[i]) {
            ty = RC.ny[i];
            // a quarter-size region: thin strips are latency-bound, so
            // spread them over 4x more CTAs
            tx = max(cap / 4 / (ty + 2 * H) - 2 * H, 8);
        } else if (RC.nx[i] < TQ) {
            tx = RC.nx[i];
            ty = max(cap / 4 / (tx + 2 * H) - 2 * H, 8);
        }
        R.y0[R.n] = RC.y0[i];
        R.x0[R.n] = RC.x0[i];
        R.ny[R.n] = RC.ny[i];
        R.nx[R.n] = RC.nx[i];
        R.ty[R.n] = ty;
        R.tx[R.n] = tx;
        const size_t c = (size_t)(ty + 2 * H) * (tx + 2 * H);
        cells = c > cells ? c : cells;
        blocks += (long)((RC.ny[i] + ty - 1) / ty) * ((RC.nx[i] + tx - 1) / tx);
        ++R.n;
    }
    if (R.n == 0) return cudaSuccess;
    const size_t smem = 2 * 4 * cells * sizeof(float);
    const dim3 grid((unsigned)blocks);
    static bool attr_set[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (!attr_set[dev & 63]) {
        const size_t maxsm = 2 * 4 * (size_t)cap * sizeof(float);
        cudaFuncSetAttribute(interp_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)maxsm);
        cudaFuncSetAttribute(interp_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)maxsm);
        attr_set[dev & 63] = true;
    }
    if (L.direction == 0)
        interp_kernel<0><<<grid, NT, smem, stream>>>(L, R);
    else
        interp_kernel<1><<<grid, NT, smem, stream>>>(L, R);
    wl_count_launch();
    return cudaGetLastError();
}

cudaError_t wl_launch_conv(const WlLevel& L, cudaStream_t stream) {
    const dim3 grid((L.qw + TQ - 1) / TQ, (L.qh + TQ - 1) / TQ);
    conv_kernel<<<grid, NT, 0, stream>>>(L);
    wl_count_launch();
    return cudaGetLastError();
}
