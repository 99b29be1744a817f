// Micro-benchmark (not product): HBM efficiency of the forward kernel's write
// pattern. Each warp writes a row segment of `seg` cells into each of 4
// planes (float2 per lane, like fast_kernel's epilogue), tiles laid out with
// stride `seg` cells; optionally it first reads the matching 2x2 pixel block
// of a 2qw x 2qh image (coalesced float4), like the forward's input stream.
//   store_pattern <qw> <seg_cells> <read:0|1>
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/sp tools/store_pattern.cu
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

__global__ void k(const float* __restrict__ img, float* p0, float* p1, float* p2, float* p3,
                  int qw, int qh, int seg, int read, int stride, int off0, int win, int vec4) {
    const int lane = threadIdx.x & 31;
    const int wid = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int nw = (gridDim.x * blockDim.x) >> 5;
    const int segs = (qw - off0) / stride;
    const int per_lane = vec4 ? 4 : 2;
    for (int job = wid; job < segs * qh; job += nw) {  // one (row, segment) per warp
        const int row = job / segs, sx = job - row * segs;
        const int s0 = off0 + sx * stride;  // segment [s0, s0 + seg)
        // win: store through aligned 64-cell windows (lanes predicated to the
        // segment) instead of lane-contiguous from s0
        const int w0 = win ? (s0 / 64) * 64 : s0;
        const int wend = win ? s0 + seg : s0 + seg;
        for (int base = w0; base < wend; base += 32 * per_lane) {
            const int c = base + per_lane * lane;
            if (c < s0 || c >= s0 + seg || c >= qw) continue;
            if (vec4) {
                float4 v4 = make_float4(c, c + 1, c + 2, c + 3);
                if (read) {
                    v4 = *reinterpret_cast<const float4*>(img + (long)(2 * row) * 2 * qw + 2 * c);
                    v4.y += img[(long)(2 * row + 1) * 2 * qw + 2 * c + 7];
                }
                const long off = (long)row * qw + c;
                *reinterpret_cast<float4*>(p0 + off) = v4;
                *reinterpret_cast<float4*>(p1 + off) = v4;
                *reinterpret_cast<float4*>(p2 + off) = v4;
                *reinterpret_cast<float4*>(p3 + off) = v4;
                continue;
            }
            float v[4][2];
            if (read) {
                const float4 e = *reinterpret_cast<const float4*>(img + (long)(2 * row) * 2 * qw + 2 * c);
                const float4 o =
                    *reinterpret_cast<const float4*>(img + (long)(2 * row + 1) * 2 * qw + 2 * c);
                v[0][0] = e.x; v[1][0] = e.y; v[0][1] = e.z; v[1][1] = e.w;
                v[2][0] = o.x; v[3][0] = o.y; v[2][1] = o.z; v[3][1] = o.w;
            } else {
                for (int q = 0; q < 4; ++q) v[q][0] = v[q][1] = (float)(c + q);
            }
            const long off = (long)row * qw + c;
            *reinterpret_cast<float2*>(p0 + off) = make_float2(v[0][0], v[0][1]);
            *reinterpret_cast<float2*>(p1 + off) = make_float2(v[1][0], v[1][1]);
            *reinterpret_cast<float2*>(p2 + off) = make_float2(v[2][0], v[2][1]);
            *reinterpret_cast<float2*>(p3 + off) = make_float2(v[3][0], v[3][1]);
        }
    }
}

int main(int argc, char** argv) {
    const int qw = atoi(argv[1]), seg = atoi(argv[2]), read = atoi(argv[3]);
    const int stride = argc > 4 ? atoi(argv[4]) : seg, off0 = argc > 5 ? atoi(argv[5]) : 0;
    const int win = argc > 6 ? atoi(argv[6]) : 0;
    const int vec4 = argc > 7 ? atoi(argv[7]) : 0;
    const int qh = qw;
    float *img, *p;
    cudaMalloc(&img, (size_t)4 * qw * qh * 4);
    cudaMalloc(&p, (size_t)4 * qw * qh * 4);
    const size_t np = (size_t)qw * qh;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float best = 1e9;
    for (int it = 0; it < 12; ++it) {
        cudaEventRecord(a);
        k<<<148 * 8, 256>>>(img, p, p + np, p + 2 * np, p + 3 * np, qw, qh, seg, read, stride,
                            off0, win, vec4);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (it >= 2 && ms < best) best = ms;
    }
    const double frac = (double)seg / stride;
    const double bytes = (double)np * 16 * (read ? 2 : 1) * frac;
    printf("vec4=%d win=%d qw=%d seg=%d stride=%d off=%d read=%d: %.4f ms  %.0f GB/s (written fraction %.3f)\n",
           vec4, win, qw, seg, stride, off0, read, best, bytes / best / 1e6, frac);
    return 0;
}
