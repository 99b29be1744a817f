// Row-strip multi-level pyramid across GPUs (BASELINE configs[3]).
//
// The reference transforms one whole Image per call (multi_level_forward,
// transform.cpp:198-227). Here one image is cut into row strips, one per rank
// (one process per GPU). Each level of a rank runs the strip transform
// (wl_dwt2_forward_strip: bit-identical rows of the whole-image transform)
// on a buffer holding its strip plus `halo` rows of each neighbour; the only
// communication is that halo, pushed every level straight into the
// neighbours' buffers over NVLink (CUDA IPC peer memory, P2P stores) and
// signalled with a release store to a flag word in the neighbour's memory
// -- no NCCL, no host round trip in the level loop.
//
// Per rank, ONE device allocation (the "window", exported by IPC handle):
//   [ level buffers l = 0..L-1: (halo + S_l + halo) x w_l floats ]
//   [ flags: per level {from_up, from_down}, then {done_up, done_down} ]
// S_l = S >> l strip rows, w_l = w >> l. Level l+1's buffer interior is the
// LL output of level l; the last level's LL goes to the caller's slice.
//
// Protocol for call (epoch) e, per rank, all in stream order:
//   0. wait until both neighbours signalled done >= e-1 (their previous call
//      finished reading the halos we are about to overwrite);
//   for l in 0..L-1:
//   1. exchange kernel: copy the top/bottom `halo` interior rows of level l
//      into the up/down neighbour's halo rows; the last CTA to finish fences
//      (system scope) and release-stores e into the neighbours' flags;
//   2. strip transform of level l. Its producer warp spins (acquire, bounded
//      by a timeout) until both of this rank's flags for level l reached e,
//      but only right before the first tile that reads a halo row; those
//      tile rows are scheduled last, so the wait overlaps the interior
//      tiles (lifting schemes, neighbours on other GPUs; otherwise -- the
//      Convolution kernel has no producer warp, and a neighbour sharing
//      this GPU could need SM room the waiting grid holds -- the exchange
//      kernel's last CTA does the wait, before the transform starts).
//   3. signal done = e to both neighbours.
// Periodic ring: rank 0's up neighbour is rank G-1. With one rank the
// neighbour is the rank itself (the wrap copies within its own buffer).
#include <unistd.h>

#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <new>
#include <string>

#include "../../include/wl_dwt.h"
#include "wl_internal.h"

namespace {

constexpr int kMaxLevels = 16;
constexpr unsigned long long kTimeoutNs = 10ull * 1000 * 1000 * 1000;  // 10 s

struct Blob {  // IPC export of a rank's window (fits WL_STRIPS_BLOB_BYTES)
    cudaIpcMemHandle_t handle;
    int pid;
    int device;
    unsigned long long ptr;  // window address in the exporting process
    unsigned long long bytes;
    unsigned char uuid[16];  // GPU identity, independent of CUDA_VISIBLE_DEVICES
};

__device__ __forceinline__ void st_release_sys(unsigned* p, unsigned v) {
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_acquire_sys(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned long long globaltimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// Spin until *a >= e and *b >= e (wrap-safe compare), or time out.
__device__ void wait_flags(const unsigned* a, const unsigned* b, unsigned e, unsigned* err) {
    const unsigned long long t0 = globaltimer();
    unsigned ns = 64;
    while ((int)(ld_acquire_sys(a) - e) < 0 || (int)(ld_acquire_sys(b) - e) < 0) {
        if (globaltimer() - t0 > kTimeoutNs) {
            atomicExch(err, 1u);
            return;
        }
        __nanosleep(ns);
        ns = ns < 1024 ? 2 * ns : 1024;
    }
}

struct XchArgs {
    const float* top;    // my first interior row
    const float* bot;    // my first row of the last `halo` interior rows
    float* up_dst;       // up neighbour: its bottom halo rows
    float* down_dst;     // down neighbour: its top halo rows
    long n;              // floats per side (halo * w_l)
    unsigned* sig_up;    // up neighbour's from_down flag
    unsigned* sig_down;  // down neighbour's from_up flag
    const unsigned* my_a;
    const unsigned* my_b;
    unsigned epoch;
    unsigned* counter;  // CTA completion counter (my window)
    unsigned* err;      // host-mapped error word
    int vec4;
    int wait;           // 1: last CTA also waits for my halos (else the transform does)
};

__global__ void __launch_bounds__(256) exchange_kernel(const XchArgs a) {
    const long stride = (long)gridDim.x * blockDim.x;
    const long i0 = (long)blockIdx.x * blockDim.x + threadIdx.x;
    if (a.vec4) {
        const long n4 = a.n / 4;
        for (long i = i0; i < n4; i += stride) {
            reinterpret_cast<float4*>(a.up_dst)[i] = reinterpret_cast<const float4*>(a.top)[i];
            reinterpret_cast<float4*>(a.down_dst)[i] = reinterpret_cast<const float4*>(a.bot)[i];
        }
    } else {
        for (long i = i0; i < a.n; i += stride) {
            a.up_dst[i] = a.top[i];
            a.down_dst[i] = a.bot[i];
        }
    }
    __threadfence_system();  // this thread's peer stores, before the count
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence_system();
        const unsigned prev = atomicAdd(a.counter, 1u);
        if (prev == gridDim.x - 1) {  // last CTA: everything above is performed
            *a.counter = 0;
            __threadfence_system();
            st_release_sys(a.sig_up, a.epoch);
            st_release_sys(a.sig_down, a.epoch);
            if (a.wait) wait_flags(a.my_a, a.my_b, a.epoch, a.err);
        }
    }
}

__global__ void signal_kernel(unsigned* sig_up, unsigned* sig_down, unsigned epoch) {
    __threadfence_system();
    st_release_sys(sig_up, epoch);
    st_release_sys(sig_down, epoch);
}

__global__ void wait_kernel(const unsigned* a, const unsigned* b, unsigned epoch, unsigned* err) {
    wait_flags(a, b, epoch, err);
}

int sfail(int code, const std::string& m) { return wl_fail(code, m.c_str()); }

}  // namespace

struct WlStrips {
    int w, rows, levels, wavelet, scheme, scaling, rank, nranks, halo, device;
    char* window = nullptr;
    size_t bytes = 0;
    size_t lvl_off[kMaxLevels];  // byte offsets of level buffers in a window
    size_t flag_off = 0;         // byte offset of the flag block
    char* up = nullptr;          // neighbours' windows (mapped)
    char* down = nullptr;
    bool up_opened = false, down_opened = false;
    bool peer_same_device = false;  // a neighbour rank (not me) lives on my GPU
    unsigned char uuid[16] = {};
    unsigned* err_host = nullptr;  // host-mapped
    unsigned* err_dev = nullptr;
    unsigned epoch = 0;

    int wl(int l) const { return w >> l; }
    int sl(int l) const { return rows >> l; }
    float* lvl(char* base, int l) const { return reinterpret_cast<float*>(base + lvl_off[l]); }
    unsigned* flags(char* base) const { return reinterpret_cast<unsigned*>(base + flag_off); }
    // flag indices: 2l = from_up[l], 2l+1 = from_down[l]; 2L = done_from_up,
    // 2L+1 = done_from_down; 2L+2 = exchange CTA counter; 2L+3, 2L+4 =
    // scratch flags of the warm-up launches (kMaxLevels = 16 -> index <= 36).
};

extern "C" {

const char* wl_strips_last_error(void) { return wl_last_error(); }

size_t wl_strips_blob_bytes(void) { return sizeof(Blob); }

int wl_strips_create(int w, int h, int rank, int nranks, int levels, int wavelet, int scheme,
                     int scaling, WlStrips** out) {
    if (!out) return sfail(WL_EINVAL, "null output");
    *out = nullptr;
    if (nranks < 1 || rank < 0 || rank >= nranks) return sfail(WL_EINVAL, "bad rank/nranks");
    if (levels < 1 || levels > kMaxLevels) return sfail(WL_EINVAL, "levels must be 1..16");
    if (wavelet < WL_CDF53 || wavelet > WL_CDF97 || scheme < 0 || scheme > 9)
        return sfail(WL_EINVAL, "strip pyramids support cdf53/cdf97 schemes");
    if (w <= 0 || h <= 0 || h % nranks != 0)
        return sfail(WL_EINVAL, "image height must split evenly into row strips");
    const int rows = h / nranks;
    const int div = 1 << levels;
    if (w % div != 0 || rows % div != 0)
        return sfail(WL_EINVAL, "strip rows and width must be divisible by 2^levels");
    const int halo = wl_strip_halo_rows(wavelet, scheme, 0);
    if ((rows >> (levels - 1)) < halo)
        return sfail(WL_EINVAL, "strip too thin for the halo at the deepest level");
    // every level's strip transform must accept its shape: checked here, before
    // any exchange kernel or flag signal of a forward call is enqueued
    for (int l = 0; l < levels; ++l)
        if (!wl_strip_shape_ok(w >> l, rows >> l, halo, wavelet, scheme, 0))
            return sfail(WL_EINVAL, "a pyramid level's shape is not supported by the strip "
                                    "kernels");
    WlStrips* s = new (std::nothrow) WlStrips();
    if (!s) return sfail(WL_ERUNTIME, "out of host memory");
    s->w = w;
    s->rows = rows;
    s->levels = levels;
    s->wavelet = wavelet;
    s->scheme = scheme;
    s->scaling = scaling;
    s->rank = rank;
    s->nranks = nranks;
    s->halo = halo;
    cudaGetDevice(&s->device);
    {
        cudaDeviceProp prop;
        if (cudaGetDeviceProperties(&prop, s->device) == cudaSuccess)
            memcpy(s->uuid, &prop.uuid, sizeof(s->uuid));
    }
    size_t off = 0;
    for (int l = 0; l < levels; ++l) {
        s->lvl_off[l] = off;
        off += static_cast<size_t>(2 * halo + s->sl(l)) * s->wl(l) * sizeof(float);
        off = (off + 255) & ~static_cast<size_t>(255);
    }
    s->flag_off = off;
    off += 256;
    s->bytes = off;
    cudaError_t e = cudaMalloc(&s->window, s->bytes);
    if (e == cudaSuccess) e = cudaMemset(s->window + s->flag_off, 0, 256);
    if (e == cudaSuccess)
        e = cudaHostAlloc(&s->err_host, sizeof(unsigned), cudaHostAllocMapped);
    if (e == cudaSuccess) {
        *s->err_host = 0;
        e = cudaHostGetDevicePointer(reinterpret_cast<void**>(&s->err_dev), s->err_host, 0);
    }
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        if (s->window) cudaFree(s->window);
        if (s->err_host) cudaFreeHost(s->err_host);
        delete s;
        return sfail(WL_ERUNTIME, std::string("wl_strips_create: ") + cudaGetErrorString(e));
    }
    if (nranks == 1) s->up = s->down = s->window;
    // Warm up every kernel the protocol launches, synchronously, BEFORE any
    // rank can spin on a neighbour: lazy module loading and the first
    // launch's cudaFuncSetAttribute synchronise the device, which would
    // deadlock a stream whose exchange kernel is waiting for a neighbour
    // whose work the host has not enqueued yet.
    {
        const int ww = 256, rr = 16;
        float* tmp = nullptr;
        const size_t img = static_cast<size_t>(rr + 2 * halo) * ww;
        const size_t np = static_cast<size_t>(ww / 2) * (rr / 2);
        e = cudaMalloc(&tmp, (img + 4 * np) * sizeof(float));
        if (e == cudaSuccess) e = cudaMemset(tmp, 0, (img + 4 * np) * sizeof(float));
        int st = WL_OK;
        if (e == cudaSuccess) {
            float* pl = tmp + img;
            st = wl_dwt2_forward_strip(tmp + static_cast<size_t>(halo) * ww, ww, rr, halo, ww,
                                       wavelet, scheme, scaling, pl, pl + np, pl + 2 * np,
                                       pl + 3 * np, ww / 2, nullptr);
            unsigned* f = s->flags(s->window);
            XchArgs a{};  // zero rows; signals and waits on scratch flags at epoch 0
            a.top = a.bot = tmp;
            a.up_dst = a.down_dst = tmp;
            a.n = 0;
            a.sig_up = f + 2 * levels + 3;
            a.sig_down = f + 2 * levels + 4;
            a.my_a = f + 2 * levels + 3;
            a.my_b = f + 2 * levels + 4;
            a.epoch = 0;
            a.counter = f + 2 * levels + 2;
            a.err = s->err_dev;
            a.wait = 1;
            exchange_kernel<<<1, 256>>>(a);
            signal_kernel<<<1, 1>>>(f + 2 * levels + 3, f + 2 * levels + 4, 0);
            wait_kernel<<<1, 1>>>(f + 2 * levels + 3, f + 2 * levels + 4, 0, s->err_dev);
            e = cudaDeviceSynchronize();
        }
        if (tmp) cudaFree(tmp);
        if (e != cudaSuccess || st != WL_OK) {
            const std::string msg = e != cudaSuccess ? std::string(cudaGetErrorString(e))
                                                     : std::string(wl_last_error());
            cudaFree(s->window);
            cudaFreeHost(s->err_host);
            delete s;
            return sfail(st != WL_OK ? st : WL_ERUNTIME, "wl_strips_create warm-up: " + msg);
        }
    }
    *out = s;
    return WL_OK;
}

int wl_strips_export(WlStrips* s, void* blob) {
    if (!s || !blob) return sfail(WL_EINVAL, "null argument");
    Blob b{};
    memset(&b, 0, sizeof(b));
    cudaError_t e = cudaIpcGetMemHandle(&b.handle, s->window);
    if (e != cudaSuccess)
        return sfail(WL_ERUNTIME, std::string("cudaIpcGetMemHandle: ") + cudaGetErrorString(e));
    b.pid = static_cast<int>(getpid());
    b.device = s->device;
    b.ptr = reinterpret_cast<unsigned long long>(s->window);
    b.bytes = s->bytes;
    memcpy(b.uuid, s->uuid, sizeof(b.uuid));
    memcpy(blob, &b, sizeof(b));
    return WL_OK;
}

// Map a neighbour's window: same process -> its pointer; else open the IPC
// handle (once per distinct handle; `other` is the already-mapped neighbour).
static int map_blob(WlStrips* s, const Blob& b, const Blob* other, char* other_ptr, char** dst,
                    bool* opened) {
    if (b.bytes != s->bytes) return sfail(WL_EINVAL, "neighbour window has a different shape");
    if (b.pid == static_cast<int>(getpid())) {
        *dst = reinterpret_cast<char*>(b.ptr);
        *opened = false;
        return WL_OK;
    }
    if (other && memcmp(&other->handle, &b.handle, sizeof(b.handle)) == 0 && other_ptr) {
        *dst = other_ptr;
        *opened = false;
        return WL_OK;
    }
    void* p = nullptr;
    cudaError_t e = cudaIpcOpenMemHandle(&p, b.handle, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess)
        return sfail(WL_ERUNTIME, std::string("cudaIpcOpenMemHandle: ") + cudaGetErrorString(e));
    *dst = static_cast<char*>(p);
    *opened = true;
    return WL_OK;
}

int wl_strips_connect(WlStrips* s, const void* up_blob, const void* down_blob) {
    if (!s || !up_blob || !down_blob) return sfail(WL_EINVAL, "null argument");
    Blob u, d;
    memcpy(&u, up_blob, sizeof(u));
    memcpy(&d, down_blob, sizeof(d));
    int st = map_blob(s, u, nullptr, nullptr, &s->up, &s->up_opened);
    if (st != WL_OK) return st;
    const unsigned long long me = reinterpret_cast<unsigned long long>(s->window);
    const int mypid = static_cast<int>(getpid());
    auto shares = [&](const Blob& b) {
        const bool self = b.pid == mypid && b.ptr == me;
        return !self && memcmp(b.uuid, s->uuid, sizeof(b.uuid)) == 0;
    };
    s->peer_same_device = shares(u) || shares(d);
    return map_blob(s, d, &u, s->up, &s->down, &s->down_opened);
}

float* wl_strips_input(WlStrips* s) {
    return s ? s->lvl(s->window, 0) + static_cast<size_t>(s->halo) * s->w : nullptr;
}

size_t wl_strips_slice_elems(const WlStrips* s) {
    return s ? static_cast<size_t>(s->rows) * s->w : 0;
}

int wl_strips_forward(WlStrips* s, float* slice, void* stream) {
    if (!s || !slice) return sfail(WL_EINVAL, "null argument");
    if (!s->up || !s->down) return sfail(WL_EINVAL, "strips not connected");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int L = s->levels, halo = s->halo;
    unsigned* my = s->flags(s->window);
    unsigned* fu = s->flags(s->up);
    unsigned* fd = s->flags(s->down);
    const unsigned e = ++s->epoch;
    // Lifting schemes: the exchange kernel only pushes and signals; the
    // strip transform's producer waits for the neighbours' halos right before
    // the tile rows that read them, which it schedules last (wl_fast_impl.cuh
    // tile_row_of), so the wait hides behind the interior tiles.
    // Only when no neighbour shares this GPU (or nranks == 1, where my own
    // exchange precedes the transform on the stream): a neighbour on the
    // same device could otherwise need SM room the waiting grid holds.
    // WL_STRIP_OVERLAP=0 disables it, =2 forces it (single-GPU tests).
    static const int overlap_env = [] {
        const char* v = getenv("WL_STRIP_OVERLAP");
        return v ? atoi(v) : 1;
    }();
    const bool overlap = wl_strip_wait_capable(s->wavelet, s->scheme) &&
                         (overlap_env == 2 || (overlap_env == 1 && !s->peer_same_device));
    if (e > 1) {  // neighbours finished reading the halos of call e-1
        wait_kernel<<<1, 1, 0, st>>>(my + 2 * L, my + 2 * L + 1, e - 1, s->err_dev);
        wl_count_launch();
    }
    size_t off = 0;
    for (int l = 0; l < L; ++l) {
        const int wl_ = s->wl(l), sl_ = s->sl(l);
        float* buf = s->lvl(s->window, l);
        float* interior = buf + static_cast<size_t>(halo) * wl_;
        XchArgs a{};
        a.top = interior;
        a.bot = interior + static_cast<size_t>(sl_ - halo) * wl_;
        a.up_dst = s->lvl(s->up, l) + static_cast<size_t>(halo + sl_) * wl_;  // its bottom halo
        a.down_dst = s->lvl(s->down, l);                                      // its top halo
        a.n = static_cast<long>(halo) * wl_;
        a.sig_up = fu + 2 * l + 1;   // I am my up neighbour's down neighbour
        a.sig_down = fd + 2 * l;     // ... and my down neighbour's up neighbour
        a.my_a = my + 2 * l;
        a.my_b = my + 2 * l + 1;
        a.epoch = e;
        a.counter = my + 2 * L + 2;
        a.err = s->err_dev;
        a.vec4 = (wl_ % 4) == 0;
        // the halo wait folds into the transform only on its TMA path
        const bool ov = overlap && wl_strip_mode(wl_, sl_, halo, s->wavelet, s->scheme, 0) == 1;
        a.wait = ov ? 0 : 1;
        const long work = a.vec4 ? a.n / 4 : a.n;
        int blocks = static_cast<int>((work + 255) / 256);
        blocks = blocks < 1 ? 1 : (blocks > 148 ? 148 : blocks);
        exchange_kernel<<<blocks, 256, 0, st>>>(a);
        wl_count_launch();
        cudaError_t ce = cudaGetLastError();
        if (ce != cudaSuccess)
            return sfail(WL_ERUNTIME, std::string("exchange_kernel: ") + cudaGetErrorString(ce));
        // level l: strip transform; LL -> next level's interior (or the slice)
        const int qw = wl_ / 2, qr = sl_ / 2;
        const size_t np = static_cast<size_t>(qw) * qr;
        float* hl = slice + off;
        off += 3 * np;
        float* ll = (l + 1 == L) ? slice + off
                                 : s->lvl(s->window, l + 1) + static_cast<size_t>(halo) * qw;
        const int r = wl_forward_strip_wait(
            interior, wl_, sl_, halo, wl_, s->wavelet, s->scheme, s->scaling, ll, hl, hl + np,
            hl + 2 * np, qw, stream, ov ? my + 2 * l : nullptr, ov ? my + 2 * l + 1 : nullptr, e,
            s->err_dev);
        if (r != WL_OK) return r;
    }
    signal_kernel<<<1, 1, 0, st>>>(fu + 2 * L + 1, fd + 2 * L, e);
    wl_count_launch();
    cudaError_t ce = cudaGetLastError();
    if (ce != cudaSuccess)
        return sfail(WL_ERUNTIME, std::string("signal_kernel: ") + cudaGetErrorString(ce));
    return WL_OK;
}

int wl_strips_check(WlStrips* s) {
    if (!s) return sfail(WL_EINVAL, "null argument");
    if (*reinterpret_cast<volatile unsigned*>(s->err_host))
        return sfail(WL_ERUNTIME, "halo exchange timed out (a neighbour rank stalled)");
    return WL_OK;
}

int wl_strips_destroy(WlStrips* s) {
    if (!s) return WL_OK;
    cudaDeviceSynchronize();
    if (s->up_opened) cudaIpcCloseMemHandle(s->up);
    if (s->down_opened) cudaIpcCloseMemHandle(s->down);
    cudaFree(s->window);
    cudaFreeHost(s->err_host);
    delete s;
    return WL_OK;
}

}  // extern "C"
