// probe_issue.cu — cycles per N16 SS MMA for different descriptor-arithmetic
// shapes in the issue loop (the conv tap loop of the fused kernels).
#include <cuda_runtime.h>
#include <cstdio>
#include "../paper_2404_03617_b200/csrc/sm100.cuh"
using namespace wl;

template <int VAR>
__global__ void k(long long* out, int iters, int Wp, int flat) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tb;
  for (int i = threadIdx.x; i < 160 * 1024 / 16; i += blockDim.x) reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  if (threadIdx.x < 32) tmem_alloc<512>(&tb);
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tb;
  if (threadIdx.x == 0) {
    const uint32_t idesc = make_idesc_f16(128, 16);
    const uint32_t a0 = smem_u32(smem), b0 = smem_u32(smem + 98304);
    const uint64_t a_base = make_sdesc(a0, flat * 16, 128);
    const uint64_t b_base = make_sdesc(b0, 128, 128);
    const uint64_t b_step = (8ull << 16) + (8ull << 32) - 8ull;
    uint64_t offA[9], offB[9];
#pragma unroll
    for (int tap = 0; tap < 9; ++tap) {
      offA[tap] = (uint64_t)((tap / 3) * Wp + tap % 3);
      offB[tap] = (uint64_t)tap * 32;
    }
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it)
      for (int t = 0; t < 2; ++t)
        for (int pr = 0; pr < 4; ++pr) {
          const uint32_t d = tmem + t * 64 + 16 * pr;
          const uint64_t ap = a_base + (uint64_t)(2 * pr * flat + t * 128);
          if (VAR == 0) {  // as in the fused kernels
            const uint64_t bp = b_base + (uint64_t)(pr * 9) * b_step;
#pragma unroll
            for (int tap = 0; tap < 9; ++tap)
              mma_ss(d, ap + (uint64_t)((tap / 3) * Wp + tap % 3), bp + (uint64_t)tap * b_step, idesc, tap > 0);
          } else if (VAR == 1) {  // precomputed per-tap deltas
            const uint64_t bp = b_base + (uint64_t)(pr * 9 * 32);
#pragma unroll
            for (int tap = 0; tap < 9; ++tap) mma_ss(d, ap + offA[tap], bp + offB[tap], idesc, tap > 0);
          } else {  // fully incremental descriptors
            uint64_t ad = ap, bd = b_base + (uint64_t)(pr * 9 * 32);
#pragma unroll
            for (int tap = 0; tap < 9; ++tap) {
              mma_ss(d, ad, bd, idesc, tap > 0);
              ad += (tap % 3 == 2) ? (uint64_t)(Wp - 2) : 1ull;
              bd += 32;
            }
          }
        }
    mma_commit(&bar);
    mbar_wait(&bar, 0);
    out[0] = clock64() - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc<512>(tmem);
}

template <int VAR>
void run(const char* what) {
  long long* d;
  cudaMalloc(&d, 8);
  auto kk = k<VAR>;
  cudaFuncSetAttribute(kk, cudaFuncAttributeMaxDynamicSharedMemorySize, 164 * 1024);
  kk<<<1, 128, 164 * 1024>>>(d, 2, 15, 296);
  kk<<<1, 128, 164 * 1024>>>(d, 200, 15, 296);
  long long h;
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("%-34s %6.2f cycles/MMA  %s\n", what, (double)h / (200 * 72), cudaGetErrorString(cudaGetLastError()));
}
int main() {
  run<0>("formula (current kernels)");
  run<1>("precomputed tap deltas");
  run<2>("incremental descriptors");
  return 0;
}
