// Probe (not product): does a TMA tensor LOAD accept a box start x that is not
// 16-byte aligned?  tma_load_check <x>
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

__global__ void k(const __grid_constant__ CUtensorMap m, int x, float* out) {
    __shared__ __align__(128) float buf[64 * 4];
    __shared__ __align__(8) uint64_t bar;
    unsigned b = (unsigned)__cvta_generic_to_shared(&bar);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(1024) : "memory");
        asm volatile(
            "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"((unsigned)__cvta_generic_to_shared(buf)),
            "l"(reinterpret_cast<uint64_t>(&m)), "r"(x), "r"(0), "r"(0), "r"(b)
            : "memory");
        asm volatile("{\n\t.reg .pred p;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n}" ::"r"(b) : "memory");
        out[0] = buf[0];
        out[1] = buf[1];
    }
}

int main(int argc, char** argv) {
    int x = atoi(argv[1]);
    using Enc = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                             CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                             CUtensorMapFloatOOBfill);
    void* fp = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
    Enc enc = reinterpret_cast<Enc>(fp);
    float h[128 * 8];
    for (int i = 0; i < 128 * 8; ++i) h[i] = i;
    float *d, *o;
    cudaMalloc(&d, sizeof(h));
    cudaMalloc(&o, 8);
    cudaMemcpy(d, h, sizeof(h), cudaMemcpyHostToDevice);
    CUtensorMap m;
    cuuint64_t dims[3] = {128, 8, 1}, str[2] = {128 * 4, 128 * 8 * 4};
    cuuint32_t box[3] = {64, 4, 1}, es[3] = {1, 1, 1};
    enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    k<<<1, 32>>>(m, x, o);
    cudaError_t e = cudaDeviceSynchronize();
    float r[2] = {-1, -1};
    cudaMemcpy(r, o, 8, cudaMemcpyDeviceToHost);
    printf("load x=%d -> %s, buf[0..1] = %g %g\n", x, cudaGetErrorString(e), r[0], r[1]);
    return 0;
}
