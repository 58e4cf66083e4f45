// probe_mma_rate.cu — cycles per tcgen05.mma (SS, kind::f16, M=128, K=16) as a
// function of N, with descriptors precomputed vs rebuilt per instruction.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o probe_rate tools/probe_mma_rate.cu
#include <cuda_runtime.h>
#include <cstdio>
#include "../paper_2404_03617_b200/csrc/sm100.cuh"
using namespace wl;

template <int N, bool PRE, int WARPS = 1>
__global__ void k_rate(long long* out, int iters) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tb;
  for (int i = threadIdx.x; i < 96 * 1024 / 16; i += blockDim.x) reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
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
  if (threadIdx.x % 32 == 0 && threadIdx.x / 32 < WARPS) {
    const int wid = threadIdx.x / 32;
    const uint32_t idesc = make_idesc_f16(128, N);
    const uint32_t a0 = smem_u32(smem), b0 = smem_u32(smem + 65536);
    uint64_t ad[8], bd[8];
    for (int i = 0; i < 8; ++i) {
      ad[i] = make_sdesc(a0 + i * 256, 2048, 128);
      bd[i] = make_sdesc(b0 + i * 256, N * 16, 128);
    }
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        if (PRE) {
          mma_ss(tmem + wid * 64, ad[k], bd[k], idesc, 1);
        } else {
          mma_ss(tmem, make_sdesc(a0 + ((it + k) & 7) * 256, 2048, 128), make_sdesc(b0 + ((it * 3 + k) & 7) * 256, N * 16, 128),
                 idesc, 1);
        }
      }
    }
    if (wid == 0) {
      mma_commit(&bar);
      mbar_wait(&bar, 0);
    }
    long long t1 = clock64();
    if (wid == 0) out[0] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc<512>(tmem);
}

template <int N, bool PRE, int WARPS = 1>
void run() {
  long long* d;
  cudaMalloc(&d, 8);
  auto k = k_rate<N, PRE, WARPS>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  const int iters = 2000;
  k<<<1, 128, 100 * 1024>>>(d, 10);
  k<<<1, 128, 100 * 1024>>>(d, iters);
  long long h;
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("N=%3d %s warps=%d: %.2f cycles per MMA (ideal %.1f)  err=%s\n", N, PRE ? "pre-built desc" : "desc per MMA  ",
         WARPS, (double)h / (iters * 8 * WARPS), 128.0 * N / 256.0, cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

int main() {
  run<16, true>();
  run<16, true, 2>();
  run<16, true, 4>();
  run<64, true, 2>();
  run<16, false>();
  run<32, true>();
  run<64, true>();
  run<64, false>();
  run<128, true>();
  run<256, true>();
  return 0;
}
