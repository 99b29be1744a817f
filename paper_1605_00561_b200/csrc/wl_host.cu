// Host-buffer entry points: the reference's own call shape (transform.hpp:
// 65-72: `forward(const Image&)` / `inverse(const QuadGrid&)` take and return
// host memory), float32 here.
//
// Large periodic cdf53/cdf97 transforms are pipelined in row chunks: chunk k
// is copied host->device (with the halo rows the strip transform needs,
// wrapped at the image border), transformed by the strip kernels
// (bit-identical rows of the whole-image transform) and copied back -- one
// stream per copy direction plus one for the kernels, chained by events per
// buffer slot, so PCIe in both directions and the kernels overlap. Every
// other case (symmetric boundary, dd137, small or unaligned images) runs
// whole-image: copy in, transform, copy out. The call returns when the
// result is in host memory. Host buffers should be pinned
// (cudaHostRegister / cudaHostAlloc) for the copies to run asynchronously.
#include <cuda_runtime.h>

#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/wl_dwt.h"
#include "wl_internal.h"

namespace {

constexpr int kMaxSlots = 8;
// pipeline depth (streams / device buffers); WL_HOST_SLOTS overrides (tuning)
int slots() {
    static const int v = [] {
        const char* e = getenv("WL_HOST_SLOTS");
        const int n = e ? atoi(e) : 3;
        return n < 2 ? 2 : (n > kMaxSlots ? kMaxSlots : n);
    }();
    return v;
}
constexpr size_t kChunkBytes = 32u << 20;  // target input bytes per chunk

struct Workspace {
    int device = -1;
    cudaStream_t streams[kMaxSlots] = {};
    cudaEvent_t done[kMaxSlots] = {};
    // chunk pipeline: one stream per copy direction and one for kernels
    // (streams[0..2]), chained per buffer slot by events
    cudaEvent_t h2d_done[kMaxSlots] = {}, k_done[kMaxSlots] = {}, d2h_done[kMaxSlots] = {};
    float* in[kMaxSlots] = {};
    float* out[kMaxSlots] = {};
    size_t in_cap = 0, out_cap = 0;  // floats per slot

    bool ensure(size_t in_floats, size_t out_floats) {
        int dev = 0;
        cudaGetDevice(&dev);
        if (device != dev) {
            release();
            device = dev;
            for (int s = 0; s < kMaxSlots; ++s) {
                if (cudaStreamCreateWithFlags(&streams[s], cudaStreamNonBlocking) != cudaSuccess)
                    return false;
                if (cudaEventCreateWithFlags(&done[s], cudaEventDisableTiming) != cudaSuccess ||
                    cudaEventCreateWithFlags(&h2d_done[s], cudaEventDisableTiming) != cudaSuccess ||
                    cudaEventCreateWithFlags(&k_done[s], cudaEventDisableTiming) != cudaSuccess ||
                    cudaEventCreateWithFlags(&d2h_done[s], cudaEventDisableTiming) != cudaSuccess)
                    return false;
            }
        }
        if (in_floats > in_cap || out_floats > out_cap) {
            free_buffers();
            const size_t ni = in_floats > in_cap ? in_floats : in_cap;
            const size_t no = out_floats > out_cap ? out_floats : out_cap;
            in_cap = out_cap = 0;
            for (int s = 0; s < slots(); ++s) {
                if (cudaMalloc(&in[s], ni * sizeof(float)) != cudaSuccess ||
                    cudaMalloc(&out[s], no * sizeof(float)) != cudaSuccess) {
                    // no half-allocated slots: the next call retries from scratch
                    free_buffers();
                    cudaGetLastError();
                    return false;
                }
            }
            in_cap = ni;  // only once every slot holds its buffers
            out_cap = no;
        }
        return true;
    }
    void free_buffers() {
        for (int s = 0; s < kMaxSlots; ++s) {
            cudaFree(in[s]);
            cudaFree(out[s]);
            in[s] = out[s] = nullptr;
        }
    }
    void release() {
        if (device < 0) return;
        for (int s = 0; s < kMaxSlots; ++s) {
            cudaFree(in[s]);
            cudaFree(out[s]);
            if (streams[s]) cudaStreamDestroy(streams[s]);
            if (done[s]) cudaEventDestroy(done[s]);
            for (cudaEvent_t* ev : {&h2d_done[s], &k_done[s], &d2h_done[s]})
                if (*ev) cudaEventDestroy(*ev), *ev = nullptr;
            in[s] = out[s] = nullptr;
            streams[s] = nullptr;
            done[s] = nullptr;
        }
        in_cap = out_cap = 0;
        device = -1;
    }
};

thread_local Workspace g_ws;

int herr(int code, const std::string& m) { return wl_fail(code, m.c_str()); }

// A failed chunk pipeline must not return while copies of earlier chunks
// still read or write the caller's (pinned) host buffers.
int drain(int code) {
    for (int k = 0; k < 3; ++k)
        if (g_ws.streams[k]) cudaStreamSynchronize(g_ws.streams[k]);
    return code;
}

int cuda_err(cudaError_t e, const char* where) {
    return herr(WL_ERUNTIME, std::string(where) + ": " + cudaGetErrorString(e));
}

// Row-block copy: one linear DMA when both sides are dense, else 2-D.
cudaError_t copy_rows(void* dst, long dpitch, const void* src, long spitch, int w, int rows,
                      cudaMemcpyKind kind, cudaStream_t s) {
    if (dpitch == w && spitch == w)
        return cudaMemcpyAsync(dst, src, static_cast<size_t>(w) * rows * 4, kind, s);
    return cudaMemcpy2DAsync(dst, dpitch * 4, src, spitch * 4, static_cast<size_t>(w) * 4, rows,
                             kind, s);
}

// Copy host rows [r0, r1) of a periodic image (rows wrap mod h) into
// consecutive device rows.
cudaError_t rows_h2d(float* dst, long dpitch, const float* src, long spitch, int w, int h, int r0,
                     int r1, cudaStream_t s) {
    int r = r0;
    while (r < r1) {
        int rr = r % h;
        rr += rr < 0 ? h : 0;
        const int n = (r1 - r) < (h - rr) ? (r1 - r) : (h - rr);
        cudaError_t e = copy_rows(dst + static_cast<long>(r - r0) * dpitch, dpitch,
                                  src + static_cast<long>(rr) * spitch, spitch, w, n,
                                  cudaMemcpyHostToDevice, s);
        if (e != cudaSuccess) return e;
        r += n;
    }
    return cudaSuccess;
}

long chunk_bytes() {
    static const long v = [] {
        const char* e = getenv("WL_HOST_CHUNK_KB");  // tuning override
        const long kb = e ? atol(e) : 0;
        return kb > 0 ? kb * 1024 : static_cast<long>(kChunkBytes);
    }();
    return v;
}

int chunk_rows(long row_bytes, int total, int align) {
    long r = chunk_bytes() / (row_bytes > 0 ? row_bytes : 1);
    r = r < 64 ? 64 : r;
    r -= r % align;
    return r >= total ? total : static_cast<int>(r);
}

// Chunk schedule over `total` rows: geometric ramp-up (R/8, R/4, R/2), steady
// chunks of ~R, ramp-down at the end -- the first chunk's H2D and the last
// chunk's D2H run without overlap, so they are kept small. Every chunk is a
// multiple of `align` rows.
std::vector<int> chunk_plan(int total, int R, int align) {
    std::vector<int> ramp;
    for (int r = R / 8; r < R; r *= 2) {
        const int rr = r - r % align;
        if (rr >= align) ramp.push_back(rr);
    }
    int rs = 0;
    for (int r : ramp) rs += r;
    std::vector<int> out;
    if (total < 2 * rs + R) {  // too small to ramp: uniform chunks
        for (int r0 = 0; r0 < total; r0 += R) out.push_back(R < total - r0 ? R : total - r0);
        return out;
    }
    out = ramp;
    const int mid = total - 2 * rs;
    const int nmid = (mid + R - 1) / R;
    int left = mid;
    for (int i = 0; i < nmid; ++i) {
        int c = left / (nmid - i);
        c -= c % align;
        if (i == nmid - 1) c = left;
        out.push_back(c);
        left -= c;
    }
    for (auto it = ramp.rbegin(); it != ramp.rend(); ++it) out.push_back(*it);
    return out;
}

// One chunk through the pipeline on buffer slot s: H2D on the copy-in
// stream (after the kernel that last read in[s]), the kernel on the compute
// stream (after this H2D and after the D2H that last read out[s]), the D2H
// on the copy-out stream. Each copy engine sees only its own direction.
template <class H, class K, class D>
int pipe_chunk(int s, H&& h2d, K&& ker, D&& d2h) {
    Workspace& w = g_ws;
    cudaStream_t si = w.streams[0], sk = w.streams[1], so = w.streams[2];
    cudaStreamWaitEvent(si, w.k_done[s], 0);
    cudaError_t e = h2d(si);
    if (e != cudaSuccess) return cuda_err(e, "H2D");
    cudaEventRecord(w.h2d_done[s], si);
    cudaStreamWaitEvent(sk, w.h2d_done[s], 0);
    cudaStreamWaitEvent(sk, w.d2h_done[s], 0);
    const int r = ker(sk);
    if (r != WL_OK) return r;
    cudaEventRecord(w.k_done[s], sk);
    cudaStreamWaitEvent(so, w.k_done[s], 0);
    e = d2h(so);
    if (e != cudaSuccess) return cuda_err(e, "D2H");
    cudaEventRecord(w.d2h_done[s], so);
    return WL_OK;
}

}  // namespace

extern "C" {

int wl_dwt2_forward_host(const float* img, int w, int h, long img_pitch, int wavelet, int scheme,
                         int boundary, int scaling, float* ll, float* hl, float* lh, float* hh,
                         long plane_pitch) {
    if (w <= 0 || h <= 0 || w % 2 != 0 || h % 2 != 0)
        return herr(WL_EINVAL, "forward requires even positive dimensions");
    if (!img || !ll || !hl || !lh || !hh) return herr(WL_EINVAL, "null buffer");
    if (img_pitch < w || plane_pitch < w / 2) return herr(WL_EINVAL, "pitch too small");
    const int qw = w / 2;
    float* hp[4] = {ll, hl, lh, hh};
    const int halo = (wavelet == WL_CDF53 || wavelet == WL_CDF97)
                         ? wl_strip_halo_rows(wavelet, scheme, 0) : -1;
    bool chunked = boundary == WL_PERIODIC && halo > 0 && h >= 2 * halo && scheme >= 0 &&
                   scheme <= 9;
    const int R = chunked ? chunk_rows(4L * w, h, 2) : h;
    // every chunk height of the plan must be a shape the strip kernels take
    if (chunked && R < h)
        for (int rows : chunk_plan(h, R, 2))
            chunked = chunked && wl_strip_shape_ok(w, rows, halo, wavelet, scheme, 0);
    if (!chunked || R >= h) {
        // whole image: one slot, copy in / transform / copy out
        const size_t nin = static_cast<size_t>(w) * h, nout = 4 * static_cast<size_t>(qw) * (h / 2);
        if (!g_ws.ensure(nin, nout)) return herr(WL_ERUNTIME, "device workspace allocation failed");
        cudaStream_t s = g_ws.streams[0];
        float* d = g_ws.in[0];
        cudaError_t e = cudaMemcpy2DAsync(d, w * 4, img, img_pitch * 4, w * 4, h,
                                          cudaMemcpyHostToDevice, s);
        if (e != cudaSuccess) return cuda_err(e, "H2D");
        const size_t np = static_cast<size_t>(qw) * (h / 2);
        float* o = g_ws.out[0];
        int st = wl_dwt2_forward(d, w, h, w, wavelet, scheme, boundary, scaling, o, o + np,
                                 o + 2 * np, o + 3 * np, qw, s);
        if (st != WL_OK) return drain(st);
        for (int c = 0; c < 4; ++c) {
            e = cudaMemcpy2DAsync(hp[c], plane_pitch * 4, o + c * np, qw * 4, qw * 4, h / 2,
                                  cudaMemcpyDeviceToHost, s);
            if (e != cudaSuccess) return drain(cuda_err(e, "D2H"));
        }
        e = cudaStreamSynchronize(s);
        return e == cudaSuccess ? WL_OK : cuda_err(e, "forward_host");
    }
    const size_t nin = static_cast<size_t>(w) * (R + 2 * halo);
    const size_t np = static_cast<size_t>(qw) * (R / 2);
    if (!g_ws.ensure(nin, 4 * np)) return herr(WL_ERUNTIME, "device workspace allocation failed");
    const std::vector<int> plan = chunk_plan(h, R, 2);
    int r0 = 0;
    for (size_t k = 0; k < plan.size(); r0 += plan[k], ++k) {
        const int s = static_cast<int>(k % slots());
        const int rows = plan[k];
        const int r1 = r0 + rows;
        float* o = g_ws.out[s];
        const size_t npc = static_cast<size_t>(qw) * (rows / 2);
        const int r = pipe_chunk(
            s,
            [&](cudaStream_t st) {
                return rows_h2d(g_ws.in[s], w, img, img_pitch, w, h, r0 - halo, r1 + halo, st);
            },
            [&](cudaStream_t st) {
                return wl_dwt2_forward_strip(g_ws.in[s] + static_cast<size_t>(halo) * w, w,
                                             rows, halo, w, wavelet, scheme, scaling, o, o + npc,
                                             o + 2 * npc, o + 3 * npc, qw, st);
            },
            [&](cudaStream_t st) {
                for (int c = 0; c < 4; ++c) {
                    const cudaError_t e =
                        copy_rows(hp[c] + static_cast<long>(r0 / 2) * plane_pitch, plane_pitch,
                                  o + c * npc, qw, qw, rows / 2, cudaMemcpyDeviceToHost, st);
                    if (e != cudaSuccess) return e;
                }
                return cudaSuccess;
            });
        if (r != WL_OK) return drain(r);
    }
    const cudaError_t e = cudaStreamSynchronize(g_ws.streams[2]);  // last D2H waits on all
    return e == cudaSuccess ? WL_OK : drain(cuda_err(e, "forward_host"));
}

int wl_dwt2_inverse_host(const float* ll, const float* hl, const float* lh, const float* hh,
                         int qw, int qh, long plane_pitch, int wavelet, int scheme, int boundary,
                         int undo_scaling, float* img, long img_pitch) {
    if (qw <= 0 || qh <= 0) return herr(WL_EINVAL, "inverse requires positive plane dimensions");
    if (!img || !ll || !hl || !lh || !hh) return herr(WL_EINVAL, "null buffer");
    if (img_pitch < 2 * qw || plane_pitch < qw) return herr(WL_EINVAL, "pitch too small");
    const float* hp[4] = {ll, hl, lh, hh};
    const int halo = (wavelet == WL_CDF53 || wavelet == WL_CDF97)
                         ? wl_strip_halo_rows(wavelet, scheme, 1) : -1;
    bool chunked = boundary == WL_PERIODIC && halo > 0 && qh >= 2 * halo && scheme >= 0 &&
                   scheme <= 9;
    const int R = chunked ? chunk_rows(16L * qw, qh, 1) : qh;
    if (chunked && R < qh)
        for (int rows : chunk_plan(qh, R, 1))
            chunked = chunked && wl_strip_shape_ok(qw, rows, halo, wavelet, scheme, 1);
    if (!chunked || R >= qh) {
        const size_t np = static_cast<size_t>(qw) * qh;
        if (!g_ws.ensure(4 * np, 4 * np))
            return herr(WL_ERUNTIME, "device workspace allocation failed");
        cudaStream_t s = g_ws.streams[0];
        float* d = g_ws.in[0];
        for (int c = 0; c < 4; ++c) {
            cudaError_t e = cudaMemcpy2DAsync(d + c * np, qw * 4, hp[c], plane_pitch * 4, qw * 4,
                                              qh, cudaMemcpyHostToDevice, s);
            if (e != cudaSuccess) return drain(cuda_err(e, "H2D"));
        }
        float* o = g_ws.out[0];
        int st = wl_dwt2_inverse(d, d + np, d + 2 * np, d + 3 * np, qw, qh, qw, wavelet, scheme,
                                 boundary, undo_scaling, o, 2 * qw, s);
        if (st != WL_OK) return drain(st);
        cudaError_t e = cudaMemcpy2DAsync(img, img_pitch * 4, o, 2 * qw * 4, 2 * qw * 4, 2 * qh,
                                          cudaMemcpyDeviceToHost, s);
        if (e != cudaSuccess) return drain(cuda_err(e, "D2H"));
        e = cudaStreamSynchronize(s);
        return e == cudaSuccess ? WL_OK : cuda_err(e, "inverse_host");
    }
    const size_t npb = static_cast<size_t>(qw) * (R + 2 * halo);  // one plane buffer
    if (!g_ws.ensure(4 * npb, static_cast<size_t>(4) * qw * R))
        return herr(WL_ERUNTIME, "device workspace allocation failed");
    const std::vector<int> plan = chunk_plan(qh, R, 1);
    int q0 = 0;
    for (size_t k = 0; k < plan.size(); q0 += plan[k], ++k) {
        const int s = static_cast<int>(k % slots());
        const int rows = plan[k];
        const int q1 = q0 + rows;
        const size_t pb = static_cast<size_t>(qw) * (rows + 2 * halo);
        float* d = g_ws.in[s] + static_cast<size_t>(halo) * qw;
        const int r = pipe_chunk(
            s,
            [&](cudaStream_t st) {
                for (int c = 0; c < 4; ++c) {
                    const cudaError_t e = rows_h2d(g_ws.in[s] + c * pb, qw, hp[c], plane_pitch, qw,
                                                   qh, q0 - halo, q1 + halo, st);
                    if (e != cudaSuccess) return e;
                }
                return cudaSuccess;
            },
            [&](cudaStream_t st) {
                return wl_dwt2_inverse_strip(d, d + pb, d + 2 * pb, d + 3 * pb, qw, rows, halo,
                                             qw, wavelet, scheme, undo_scaling, g_ws.out[s],
                                             2 * qw, st);
            },
            [&](cudaStream_t st) {
                return copy_rows(img + static_cast<long>(2 * q0) * img_pitch, img_pitch,
                                 g_ws.out[s], 2 * qw, 2 * qw, 2 * rows, cudaMemcpyDeviceToHost,
                                 st);
            });
        if (r != WL_OK) return drain(r);
    }
    const cudaError_t e = cudaStreamSynchronize(g_ws.streams[2]);  // last D2H waits on all
    return e == cudaSuccess ? WL_OK : drain(cuda_err(e, "inverse_host"));
}

}  // extern "C"
