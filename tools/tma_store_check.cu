// Standalone probe of TMA tensor stores (not product). One case per process:
//   tma_store_check <box_h> <x> <y> <smem_off_floats> <nmaps_in_struct> <sel> <W> <H>
// nvcc -gencode arch=compute_100a,code=sm_100a -o tools/tma_store_check tools/tma_store_check.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

struct Maps { CUtensorMap m[8]; };

__device__ __forceinline__ unsigned su32(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}

__global__ void k(const __grid_constant__ Maps mm, int x, int y, int sel, int off) {
    extern __shared__ __align__(128) float buf[];
    for (int i = threadIdx.x; i < off + 60 * 16; i += blockDim.x) buf[i] = i;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile(
            "cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
                reinterpret_cast<uint64_t>(&mm.m[sel])),
            "r"(su32(buf + off)), "r"(x), "r"(y), "r"(0)
            : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }
}

int main(int argc, char** argv) {
    int bh = atoi(argv[1]), x = atoi(argv[2]), y = atoi(argv[3]), off = atoi(argv[4]);
    int sel = atoi(argv[6]), W = atoi(argv[7]), Hh = atoi(argv[8]);
    using Enc = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                             CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                             CUtensorMapFloatOOBfill);
    void* fp = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
    Enc enc = reinterpret_cast<Enc>(fp);
    float* d;
    cudaMalloc(&d, (size_t)W * Hh * 4);
    Maps mm;
    for (int s = 0; s < 8; ++s) {
        cuuint64_t dims[3] = {(cuuint64_t)W, (cuuint64_t)Hh, 1},
                   str[2] = {(cuuint64_t)W * 4, (cuuint64_t)W * Hh * 4};
        cuuint32_t box[3] = {60, (cuuint32_t)bh, 1}, es[3] = {1, 1, 1};
        CUresult r = enc(&mm.m[s], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, d, dims, str, box, es,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r) printf("encode fail %d\n", (int)r);
    }
    size_t smem = (off + 60 * 16) * 4;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k<<<1, 128, smem>>>(mm, x, y, sel, off);
    cudaError_t e = cudaDeviceSynchronize();
    printf("bh=%d x=%d y=%d off=%d sel=%d W=%d H=%d -> %s\n", bh, x, y, off, sel, W, Hh,
           cudaGetErrorString(e));
    return e != cudaSuccess;
}
