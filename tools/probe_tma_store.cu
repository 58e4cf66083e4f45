// probe_tma_store.cu — which TMA stores of a 128B-swizzled smem tile are legal:
// (a) box start at a negative coordinate (OOB columns dropped?)
// (b) box start 0 with the smem source 128 B past a 1024-aligned base
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/probe_tma_store tools/probe_tma_store.cu -lcuda
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <vector>
#include "../paper_2404_03617_b200/csrc/sm100.cuh"
using namespace wl;

__global__ void k_store(const __grid_constant__ CUtensorMap tm, int mode) {
  extern __shared__ __align__(1024) uint8_t smem[];
  // rows of 128 B (64 fp16): row r chunk c holds value r*100 + c (in the swizzled position)
  for (int i = threadIdx.x; i < 32 * 8; i += blockDim.x) {
    const int r = i / 8, c = i % 8;
    __half v = __float2half((float)(r * 100 + c));
    uint4 q;
    __half2 h2 = __halves2half2(v, v);
    q.x = q.y = q.z = q.w = *reinterpret_cast<uint32_t*>(&h2);
    *reinterpret_cast<uint4*>(smem + r * 128 + ((c ^ (r & 7)) << 4)) = q;
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint8_t* src = mode == 0 ? smem : smem + 128;
    const int x0 = mode == 0 ? -1 : 0;
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(&tm),
                 "r"(smem_u32(src)), "r"(0), "r"(x0)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
}

typedef CUresult (*PFN_t)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                          const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  void* fn;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  PFN_t enc = (PFN_t)fn;
  const int W = 14;  // valid columns
  __half* d;
  cudaMalloc(&d, 64 * 64 * 2);
  for (int mode = 1; mode >= 0; --mode) {
    cudaMemset(d, 0, 64 * 64 * 2);
    CUtensorMap tm;
    cuuint64_t dims[2] = {64, (cuuint64_t)W};
    cuuint64_t str[1] = {128};
    cuuint32_t box[2] = {64, 16}, es[2] = {1, 1};
    enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    cudaFuncSetAttribute(k_store, cudaFuncAttributeMaxDynamicSharedMemorySize, 8192);
    k_store<<<1, 128, 8192>>>(tm, mode);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<__half> h(64 * W);
    cudaMemcpy(h.data(), d, 64 * W * 2, cudaMemcpyDeviceToHost);
    printf("mode %d (%s): %s; row0 chunk0..7 =", mode, mode == 0 ? "x0=-1" : "src+128B, x0=0", cudaGetErrorString(e));
    for (int c = 0; c < 8; ++c) printf(" %.0f", __half2float(h[c * 8]));
    printf(" | row13 chunk0 = %.0f\n", __half2float(h[13 * 64]));
    if (e != cudaSuccess) {
      cudaDeviceReset();
      cudaMalloc(&d, 64 * 64 * 2);
    }
  }
  return 0;
}
