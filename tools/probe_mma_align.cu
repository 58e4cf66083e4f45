// probe_mma_align.cu — cycles per tcgen05.mma (kind::f16, M=128, K=16) for
// SS with A start aligned / misaligned to the 128-byte core matrix, SS with
// the conv's LBO/SBO, and TS (A from TMEM), as a function of N.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o probe_align tools/probe_mma_align.cu
#include <cuda_runtime.h>
#include <cstdio>
#include "../paper_2404_03617_b200/csrc/sm100.cuh"
using namespace wl;

// MODE 0: SS, A offsets (k*256 + AOFF); MODE 1: TS
template <int N, int MODE, int AOFF, int LBO, int ND = 1, int M = 128>
__global__ void k_rate(long long* out, int iters) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tb;
  for (int i = threadIdx.x; i < 160 * 1024 / 16; i += blockDim.x) reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  if (threadIdx.x < 32) tmem_alloc<512>(&tb);
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tb;
  if (threadIdx.x == 0) {
    const uint32_t idesc = make_idesc_f16(M, N);
    const uint32_t a0 = smem_u32(smem), b0 = smem_u32(smem + 131072);
    uint64_t ad[8], bd[8];
    for (int i = 0; i < 8; ++i) {
      ad[i] = make_sdesc(a0 + i * 256 + AOFF, LBO, 128);
      bd[i] = make_sdesc(b0 + i * 256, N * 16, 128);
    }
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const uint32_t dcol = tmem + 256 + (k % ND) * N;
        if (MODE == 0) mma_ss(dcol, ad[k], bd[k], idesc, 1);
        else mma_ts(dcol, tmem + k * 8, bd[k], idesc, 1);
      }
    }
    mma_commit(&bar);
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    out[0] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc<512>(tmem);
}

template <int N, int MODE, int AOFF, int LBO, int ND = 1, int M = 128>
void run(const char* what) {
  long long* d;
  cudaMalloc(&d, 8);
  auto k = k_rate<N, MODE, AOFF, LBO, ND, M>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 164 * 1024);
  const int iters = 2000;
  k<<<1, 128, 164 * 1024>>>(d, 10);
  k<<<1, 128, 164 * 1024>>>(d, iters);
  long long h;
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("%-34s M=%d ND=%d N=%3d: %6.2f cycles/MMA (compute floor %5.1f)  %s\n", what, M, ND, N, (double)h / (iters * 8),
         128.0 * N / 256.0, cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

int main() {
  run<16, 0, 0, 2048, 1, 128>("SS");
  run<16, 0, 0, 2048, 1, 64>("SS");
  run<16, 0, 0, 2048, 4, 64>("SS");
  run<32, 0, 0, 2048, 1, 64>("SS");
  run<64, 0, 0, 2048, 1, 64>("SS");
  run<128, 0, 0, 2048, 1, 64>("SS");
  run<256, 0, 0, 2048, 1, 64>("SS");
  run<16, 1, 0, 0, 1, 64>("TS");
  run<64, 1, 0, 0, 1, 64>("TS");
  return 0;
}
