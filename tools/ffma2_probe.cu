// FP32 issue-rate probe for the stencil kernels (run on the GPU box):
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ffma2_probe tools/ffma2_probe.cu
// Measures FMA lanes/clk/SM for scalar FFMA with an immediate coefficient, packed FFMA2
// (fma.rn.f32x2, immediate broadcast coefficient), and each mixed with ALU work, so the
// lifting/polyphase/convolution generators know what one packed FMA costs in issue slots.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned long long pk(float a, float b) {
    unsigned long long r; asm("mov.b64 %0, {%1,%2};" : "=l"(r) : "f"(a), "f"(b)); return r;
}
__device__ __forceinline__ float2 upk(unsigned long long r) {
    float2 f; asm("mov.b64 {%0,%1}, %2;" : "=f"(f.x), "=f"(f.y) : "l"(r)); return f;
}
__device__ __forceinline__ unsigned long long fma2(unsigned long long a, float c, unsigned long long b) {
    unsigned long long d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(pk(c, c)), "l"(b));
    return d;
}

__device__ __forceinline__ float fma1(float a, float c, float b) {  // kept scalar (no auto-pairing)
    float d; asm("fma.rn.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(c), "f"(b)); return d;
}

constexpr int CH = 8;  // independent chains per thread

template <int MODE>
__global__ void probe(float* out, float seed, int iters) {
    float a[CH], b[CH];
    unsigned long long p[CH], q[CH];
    unsigned ia = threadIdx.x, ib = blockIdx.x;
#pragma unroll
    for (int c = 0; c < CH; ++c) {
        a[c] = seed + c; b[c] = seed - c;
        p[c] = pk(a[c], b[c]); q[c] = pk(b[c], a[c]);
    }
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
#pragma unroll
            for (int c = 0; c < CH; ++c) {
                if (MODE == 0 || MODE == 2) {           // 2 scalar FFMA (imm) = 2 FMAs
                    a[c] = fma1(a[c], 0.99951171875f, b[c]);
                    b[c] = fma1(b[c], -0.7109375f, a[c]);
                } else {                                // 1 FFMA2 (imm) = 2 FMAs
                    p[c] = fma2(p[c], 0.99951171875f, q[c]);
                }
                if (MODE == 2 || MODE == 3) {           // + 1 ALU op per 2 (scalar) or 4 (packed) FMAs
                    ia = (ia ^ (ib + c)) + 0x9e3779b9u;
                }
            }
            if (MODE == 1 || MODE == 3) {
#pragma unroll
                for (int c = 0; c < CH; ++c) q[c] = fma2(q[c], -0.7109375f, p[c]);
            }
        }
    }
    float s = 0.f;
#pragma unroll
    for (int c = 0; c < CH; ++c) {
        float2 f = upk(p[c]), g = upk(q[c]);
        s += a[c] + b[c] + f.x + f.y + g.x + g.y;
    }
    if (s == 12345.f || ia == 7u) out[blockIdx.x * blockDim.x + threadIdx.x] = s + ia;
}

int main() {
    int sms = 0, clk = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    float* out; cudaMalloc(&out, 1 << 24);
    const int threads = 256, iters = 4096;
    const char* names[4] = {"FFMA imm", "FFMA2 imm", "FFMA imm + ALU", "FFMA2 imm + ALU"};
    for (int bps : {1, 2, 4}) {
        int blocks = sms * bps;
        for (int mode = 0; mode < 4; ++mode) {
            cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
            float best = 1e30f;
            for (int rep = 0; rep < 5; ++rep) {
                cudaEventRecord(e0);
                switch (mode) {
                    case 0: probe<0><<<blocks, threads>>>(out, 1.f, iters); break;
                    case 1: probe<1><<<blocks, threads>>>(out, 1.f, iters); break;
                    case 2: probe<2><<<blocks, threads>>>(out, 1.f, iters); break;
                    case 3: probe<3><<<blocks, threads>>>(out, 1.f, iters); break;
                }
                cudaEventRecord(e1); cudaEventSynchronize(e1);
                float ms; cudaEventElapsedTime(&ms, e0, e1);
                if (ms < best) best = ms;
            }
            double fmas = double(blocks) * threads * iters * 4 * CH * ((mode & 1) ? 4 : 2);
            double tf = fmas / (best * 1e-3) / 1e12;
            // lanes/clk/SM at the nominal max clock (the box runs near it under this load)
            double per_clk = fmas / (best * 1e-3) / (double(clk) * 1e3) / sms;
            printf("warps/SM %2d  %-16s %8.3f ms  %6.2f TFMA/s  %6.1f FMA lanes/clk/SM (at %d MHz)\n",
                   bps * threads / 32, names[mode], best, tf, per_clk, clk / 1000);
        }
    }
    cudaError_t e = cudaGetLastError();
    printf("status: %s\n", cudaGetErrorString(e));
    return 0;
}
