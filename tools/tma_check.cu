// Debug probe (not product): TMA descriptor addressing variants.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
typedef CUresult (*Enc)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
__device__ __forceinline__ void tma(unsigned d, const CUtensorMap* m, unsigned b, int x, int y) {
  asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
    :: "r"(d), "l"((uint64_t)m), "r"(x), "r"(y), "r"(b) : "memory");
}
struct Args { float* out; int x, y, mode; };
__global__ void k4(const __grid_constant__ CUtensorMap m0, const __grid_constant__ CUtensorMap m1, const Args a) {
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t* bar = (uint64_t*)(sm + 4 * 8704);
  unsigned b = (unsigned)__cvta_generic_to_shared(bar);
  unsigned d = (unsigned)__cvta_generic_to_shared(sm);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(b));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    int n = (a.mode == 6) ? 2 : 1;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(b), "r"(n * 8704) : "memory");
    switch (a.mode) {
      case 4: tma(d, &m0, b, 0, 0); break;
      case 5: tma(d, &m1, b, 0, 0); break;
      case 6: tma(d, &m0, b, 0, 0); tma(d + 8704, &m0, b, 0, 0); break;
      case 7: tma(d, &m0, b, a.x, a.y); break;
      case 8: tma(d + 8704, &m0, b, 0, 0); break;
    }
    asm volatile("{\n.reg .pred p;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}" :: "r"(b) : "memory");
    a.out[0] = ((float*)sm)[0];
  }
}
int main(int argc, char** argv) {
  int mode = atoi(argv[1]);
  void* p; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  Enc enc = (Enc)p;
  float* g; cudaMalloc(&g, 4 * 128 * 128 * 4);
  float* out; cudaMalloc(&out, 64);
  CUtensorMap m[2];
  for (int i = 0; i < 2; ++i) {
    cuuint64_t dims[2] = {128, 128}; cuuint64_t str[1] = {512};
    cuuint32_t box[2] = {64, 34}; cuuint32_t es[2] = {1, 1};
    enc(&m[i], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, g + i * 128 * 128, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  Args a{out, 62, 90, mode};
  cudaFuncSetAttribute(k4, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000);
  k4<<<1, 32, 4 * 8704 + 64>>>(m[0], m[1], a);
  printf("mode %d: %s\n", mode, cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
