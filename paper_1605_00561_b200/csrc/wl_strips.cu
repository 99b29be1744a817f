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
// Symmetric boundary: no ring -- rank 0 has no upper and rank G-1 no lower
// neighbour; their transforms start/end at the image edge (0 halo rows there,
// per-step mirroring exactly as the whole image), the missing side's pushes
// are skipped and its signals/waits go to a self flag the rank sets itself.
//
// Inverse (multi_level_inverse, transform.cpp:229-256) of a slice laid out as
// the forward's: coarsest level first; per level the rank's LL rows (the
// previous level's output, or the slice's coarsest LL) and its detail rows
// (copied from the slice) sit in 4 halo-padded plane buffers of the window;
// the exchange kernel pushes `halo_q` rows of all 4 planes to each
// neighbour, then the inverse strip transform writes the next level's LL
// rows (or, at level 0, the caller's image rows).
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
    int push_up, push_down;  // 0: no neighbour on that side (symmetric image edge)
    int planes;         // blocks to push per side (4 plane buffers for the inverse)
    long plane_stride;  // floats between the blocks of consecutive planes
};

__global__ void __launch_bounds__(256) exchange_kernel(const XchArgs a) {
    const long stride = (long)gridDim.x * blockDim.x;
    const long i0 = (long)blockIdx.x * blockDim.x + threadIdx.x;
    for (int k = 0; k < a.planes; ++k) {
        const long o = k * a.plane_stride;
        if (a.vec4) {
            const long n4 = a.n / 4;
            for (long i = i0; i < n4; i += stride) {
                if (a.push_up)
                    reinterpret_cast<float4*>(a.up_dst + o)[i] =
                        reinterpret_cast<const float4*>(a.top + o)[i];
                if (a.push_down)
                    reinterpret_cast<float4*>(a.down_dst + o)[i] =
                        reinterpret_cast<const float4*>(a.bot + o)[i];
            }
        } else {
            for (long i = i0; i < a.n; i += stride) {
                if (a.push_up) a.up_dst[o + i] = a.top[o + i];
                if (a.push_down) a.down_dst[o + i] = a.bot[o + i];
            }
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
    int boundary = WL_PERIODIC;
    int halo_q = 0;               // inverse: plane rows pushed per side
    char* window = nullptr;
    size_t bytes = 0;
    size_t lvl_off[kMaxLevels];  // byte offsets of level buffers in a window
    size_t inv_off[kMaxLevels];  // byte offsets of the inverse's 4-plane buffers
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
    // symmetric: is there a neighbour above / below (else: the image edge)
    bool has_up() const { return boundary == WL_PERIODIC || rank > 0; }
    bool has_down() const { return boundary == WL_PERIODIC || rank < nranks - 1; }
    // inverse level l: plane k (LL, HL, LH, HH) of (wl/2) x (halo_q + sl/2 + halo_q)
    long inv_plane_floats(int l) const {
        return static_cast<long>(wl(l) / 2) * (sl(l) / 2 + 2 * halo_q);
    }
    float* inv_plane(char* base, int l, int k) const {
        return reinterpret_cast<float*>(base + inv_off[l]) + k * inv_plane_floats(l);
    }
    float* inv_interior(char* base, int l, int k) const {
        return inv_plane(base, l, k) + static_cast<long>(halo_q) * (wl(l) / 2);
    }
    // flag indices: 2l = from_up[l], 2l+1 = from_down[l]; 2L = done_from_up,
    // 2L+1 = done_from_down; 2L+2 = exchange CTA counter; 2L+3, 2L+4 =
    // scratch flags of the warm-up launches; 2L+5 = self flag (symmetric
    // image edge: the missing neighbour's signals and waits) (kMaxLevels =
    // 16 -> index <= 37).
};

namespace {

// Level l of the forward pyramid: the strip transform of the level buffer
// (halo rows on the sides that have a neighbour), waiting for the
// neighbours' halo flags inside the transform when xa/xb are given.
int level_forward(WlStrips* s, int l, float* ll, float* hl, float* lh, float* hh, void* stream,
                  const unsigned* xa, const unsigned* xb, unsigned e) {
    const int w_ = s->wl(l), r_ = s->sl(l);
    float* interior = s->lvl(s->window, l) + static_cast<size_t>(s->halo) * w_;
    return wl_forward_strip_wait(interior, w_, r_, s->halo, w_, s->wavelet, s->scheme, s->scaling,
                                 ll, hl, lh, hh, w_ / 2, stream, xa, xb, e, s->err_dev,
                                 s->boundary, s->has_up() ? s->halo : 0,
                                 s->has_down() ? s->halo : 0);
}

// Level l of the inverse pyramid: the 4 halo-padded plane buffers -> the
// level's input rows (w_l x s_l), at `out` with pitch `out_pitch`.
int level_inverse(WlStrips* s, int l, float* out, long out_pitch, void* stream) {
    const int qw = s->wl(l) / 2, qr = s->sl(l) / 2;
    return wl_inverse_strip_ex(s->inv_interior(s->window, l, 0), s->inv_interior(s->window, l, 1),
                               s->inv_interior(s->window, l, 2), s->inv_interior(s->window, l, 3),
                               qw, qr, s->has_up() ? s->halo_q : 0,
                               s->has_down() ? s->halo_q : 0, qw, s->wavelet, s->scheme,
                               s->scaling, out, out_pitch, stream, s->boundary);
}

}  // namespace

extern "C" {

const char* wl_strips_last_error(void) { return wl_last_error(); }

size_t wl_strips_blob_bytes(void) { return sizeof(Blob); }

int wl_strips_create(int w, int h, int rank, int nranks, int levels, int wavelet, int scheme,
                     int scaling, WlStrips** out) {
    return wl_strips_create_ex(w, h, rank, nranks, levels, wavelet, scheme, WL_PERIODIC, scaling,
                               out);
}

int wl_strips_create_ex(int w, int h, int rank, int nranks, int levels, int wavelet, int scheme,
                        int boundary, int scaling, WlStrips** out) {
    if (!out) return sfail(WL_EINVAL, "null output");
    if (boundary != WL_PERIODIC && boundary != WL_SYMMETRIC)
        return sfail(WL_EINVAL, "unknown boundary");
    if (boundary == WL_SYMMETRIC && scheme == WL_CONVOLUTION)
        return sfail(WL_EINVAL, "symmetric strip pyramids need a lifting scheme");
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
    const bool sym = boundary == WL_SYMMETRIC;
    const int ht = sym && rank == 0 ? 0 : halo, hb = sym && rank == nranks - 1 ? 0 : halo;
    const int hq = wl_strip_halo_rows(wavelet, scheme, 1);
    const int iht = sym && rank == 0 ? 0 : hq, ihb = sym && rank == nranks - 1 ? 0 : hq;
    for (int l = 0; l < levels; ++l)
        if (!wl_strip_mode_b(w >> l, rows >> l, ht, hb, wavelet, scheme, 0, boundary) ||
            !wl_strip_mode_b((w >> l) / 2, (rows >> l) / 2, iht, ihb, wavelet, scheme, 1,
                             boundary))
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
    s->boundary = boundary;
    s->halo_q = hq;
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
    for (int l = 0; l < levels; ++l) {
        s->inv_off[l] = off;
        off += 4 * static_cast<size_t>(s->inv_plane_floats(l)) * sizeof(float);
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
            (void)np;
            // every level's forward and inverse transform at its real shape
            // (hits exactly the kernel variants the calls use), on scratch
            // contents of the window
            for (int l = 0; l < levels && st == WL_OK; ++l) {
                st = level_forward(s, l, s->inv_interior(s->window, l, 0),
                                   s->inv_interior(s->window, l, 1),
                                   s->inv_interior(s->window, l, 2),
                                   s->inv_interior(s->window, l, 3), nullptr, nullptr, nullptr, 0);
                if (st == WL_OK)
                    st = level_inverse(s, l, s->lvl(s->window, l) +
                                                 static_cast<size_t>(halo) * s->wl(l),
                                       s->wl(l), nullptr);
            }
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

}  // extern "C"

namespace {

// Flag words of one call: where my signals to the up/down neighbour go and
// which of my words I wait on -- the self flag on a symmetric image edge.
struct Flags {
    unsigned *my, *fu, *fd, *self;
    int L;
    unsigned* sig_up(const WlStrips* s, int i) const { return s->has_up() ? fu + i : self; }
    unsigned* sig_down(const WlStrips* s, int i) const { return s->has_down() ? fd + i : self; }
    unsigned* from_up(const WlStrips* s, int i) const { return s->has_up() ? my + i : self; }
    unsigned* from_down(const WlStrips* s, int i) const { return s->has_down() ? my + i : self; }
};

Flags call_flags(WlStrips* s) {
    Flags f;
    f.L = s->levels;
    f.my = s->flags(s->window);
    f.fu = s->flags(s->up);
    f.fd = s->flags(s->down);
    f.self = f.my + 2 * s->levels + 5;
    return f;
}

// Overlap of the halo wait with the transform (lifting schemes, neighbours
// on other GPUs). WL_STRIP_OVERLAP=0 disables it, =2 forces it (tests).
bool overlap_ok(const WlStrips* s) {
    static const int overlap_env = [] {
        const char* v = getenv("WL_STRIP_OVERLAP");
        return v ? atoi(v) : 1;
    }();
    return wl_strip_wait_capable(s->wavelet, s->scheme) &&
           (overlap_env == 2 || (overlap_env == 1 && !s->peer_same_device));
}

int start_call(WlStrips* s, const Flags& f, unsigned e, cudaStream_t st) {
    // the self flag carries this call's epoch for the missing side's waits
    if (!s->has_up() || !s->has_down()) {
        signal_kernel<<<1, 1, 0, st>>>(f.self, f.self, e);
        wl_count_launch();
    }
    if (e > 1) {  // neighbours finished reading the halos of call e-1
        wait_kernel<<<1, 1, 0, st>>>(f.from_up(s, 2 * f.L), f.from_down(s, 2 * f.L + 1), e - 1,
                                     s->err_dev);
        wl_count_launch();
    }
    const cudaError_t ce = cudaGetLastError();
    return ce == cudaSuccess ? WL_OK
                             : sfail(WL_ERUNTIME, std::string("strips: ") + cudaGetErrorString(ce));
}

// Push `rows` rows (of `w_` floats) x `planes` plane blocks from my top /
// bottom interior into the up / down neighbour's bottom / top halo, signal
// level flag pair `i`; wait == 1: the last CTA also waits for my halos.
int exchange(WlStrips* s, const Flags& f, int i, unsigned e, const float* top, const float* bot,
             float* up_dst, float* down_dst, long n, int w_, int planes, long plane_stride,
             bool wait, cudaStream_t st) {
    XchArgs a{};
    a.top = top;
    a.bot = bot;
    a.up_dst = up_dst;
    a.down_dst = down_dst;
    a.n = n;
    a.push_up = s->has_up();
    a.push_down = s->has_down();
    a.planes = planes;
    a.plane_stride = plane_stride;
    a.sig_up = f.sig_up(s, i + 1);    // I am my up neighbour's down neighbour
    a.sig_down = f.sig_down(s, i);    // ... and my down neighbour's up neighbour
    a.my_a = f.from_up(s, i);
    a.my_b = f.from_down(s, i + 1);
    a.epoch = e;
    a.counter = f.my + 2 * f.L + 2;
    a.err = s->err_dev;
    a.vec4 = (w_ % 4) == 0 && (plane_stride % 4) == 0;
    a.wait = wait ? 1 : 0;
    const long work = (a.vec4 ? n / 4 : n) * planes;
    int blocks = static_cast<int>((work + 255) / 256);
    blocks = blocks < 1 ? 1 : (blocks > 148 ? 148 : blocks);
    exchange_kernel<<<blocks, 256, 0, st>>>(a);
    wl_count_launch();
    const cudaError_t ce = cudaGetLastError();
    return ce == cudaSuccess
               ? WL_OK
               : sfail(WL_ERUNTIME, std::string("exchange_kernel: ") + cudaGetErrorString(ce));
}

int end_call(WlStrips* s, const Flags& f, unsigned e, cudaStream_t st) {
    signal_kernel<<<1, 1, 0, st>>>(f.sig_up(s, 2 * f.L + 1), f.sig_down(s, 2 * f.L), e);
    wl_count_launch();
    const cudaError_t ce = cudaGetLastError();
    return ce == cudaSuccess
               ? WL_OK
               : sfail(WL_ERUNTIME, std::string("signal_kernel: ") + cudaGetErrorString(ce));
}

}  // namespace

extern "C" {

int wl_strips_forward(WlStrips* s, float* slice, void* stream) {
    if (!s || !slice) return sfail(WL_EINVAL, "null argument");
    if (!s->up || !s->down) return sfail(WL_EINVAL, "strips not connected");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int L = s->levels, halo = s->halo;
    const Flags f = call_flags(s);
    const unsigned e = ++s->epoch;
    // Lifting schemes: the exchange kernel only pushes and signals; the
    // strip transform's producer waits for the neighbours' halos right before
    // the tile rows that read them, which it schedules last (wl_fast_impl.cuh
    // tile_row_of), so the wait hides behind the interior tiles -- only when
    // no neighbour shares this GPU: a neighbour on the same device could
    // otherwise need SM room the waiting grid holds.
    const bool overlap = overlap_ok(s);
    int r = start_call(s, f, e, st);
    if (r != WL_OK) return r;
    size_t off = 0;
    for (int l = 0; l < L; ++l) {
        const int wl_ = s->wl(l), sl_ = s->sl(l);
        float* interior = s->lvl(s->window, l) + static_cast<size_t>(halo) * wl_;
        // the halo wait folds into the transform only on its TMA path
        const bool ov = overlap && wl_strip_mode_b(wl_, sl_, s->has_up() ? halo : 0,
                                                   s->has_down() ? halo : 0, s->wavelet,
                                                   s->scheme, 0, s->boundary) == 1;
        r = exchange(s, f, 2 * l, e, interior, interior + static_cast<size_t>(sl_ - halo) * wl_,
                     s->lvl(s->up, l) + static_cast<size_t>(halo + sl_) * wl_,  // its bottom halo
                     s->lvl(s->down, l),                                        // its top halo
                     static_cast<long>(halo) * wl_, wl_, 1, 0, !ov, st);
        if (r != WL_OK) return r;
        // level l: strip transform; LL -> next level's interior (or the slice)
        const int qw = wl_ / 2, qr = sl_ / 2;
        const size_t np = static_cast<size_t>(qw) * qr;
        float* hl = slice + off;
        off += 3 * np;
        float* ll = (l + 1 == L) ? slice + off
                                 : s->lvl(s->window, l + 1) + static_cast<size_t>(halo) * qw;
        r = level_forward(s, l, ll, hl, hl + np, hl + 2 * np, stream,
                          ov ? f.from_up(s, 2 * l) : nullptr, ov ? f.from_down(s, 2 * l + 1) : nullptr,
                          e);
        if (r != WL_OK) return r;
    }
    return end_call(s, f, e, st);
}

int wl_strips_inverse(WlStrips* s, const float* slice, float* out_rows, void* stream) {
    if (!s || !slice || !out_rows) return sfail(WL_EINVAL, "null argument");
    if (!s->up || !s->down) return sfail(WL_EINVAL, "strips not connected");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int L = s->levels, hq = s->halo_q;
    const Flags f = call_flags(s);
    const unsigned e = ++s->epoch;
    int r = start_call(s, f, e, st);
    if (r != WL_OK) return r;
    size_t offs[kMaxLevels + 1];
    size_t off = 0;
    for (int l = 0; l < L; ++l) {
        offs[l] = off;
        off += 3 * static_cast<size_t>(s->wl(l) / 2) * (s->sl(l) / 2);
    }
    offs[L] = off;  // coarsest LL
    for (int l = L - 1; l >= 0; --l) {
        const int qw = s->wl(l) / 2, qr = s->sl(l) / 2;
        const size_t np = static_cast<size_t>(qw) * qr;
        // this level's detail rows (and, at the coarsest level, LL) from the slice
        for (int k = (l == L - 1 ? 0 : 1); k < 4; ++k) {
            const float* src = k == 0 ? slice + offs[L] : slice + offs[l] + (k - 1) * np;
            const cudaError_t ce = cudaMemcpyAsync(s->inv_interior(s->window, l, k), src,
                                                   np * sizeof(float),
                                                   cudaMemcpyDeviceToDevice, st);
            if (ce != cudaSuccess)
                return sfail(WL_ERUNTIME, std::string("strips inverse copy: ") +
                                              cudaGetErrorString(ce));
        }
        const long pf = s->inv_plane_floats(l);
        r = exchange(s, f, 2 * l, e, s->inv_interior(s->window, l, 0),
                     s->inv_interior(s->window, l, 0) + static_cast<long>(qr - hq) * qw,
                     s->inv_plane(s->up, l, 0) + static_cast<long>(hq + qr) * qw,
                     s->inv_plane(s->down, l, 0), static_cast<long>(hq) * qw, qw, 4, pf, true,
                     st);
        if (r != WL_OK) return r;
        // level l inverse: its input rows = LL of level l-1 (or the image)
        float* out = l == 0 ? out_rows : s->inv_interior(s->window, l - 1, 0);
        r = level_inverse(s, l, out, 2 * qw, stream);
        if (r != WL_OK) return r;
    }
    return end_call(s, f, e, st);
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
