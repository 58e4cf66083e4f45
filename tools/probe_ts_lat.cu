// probe_ts_lat.cu — latency of one MBConv expansion (2 tiles x 8 K-steps,
// M=128, N=HC) from first issue to mbarrier completion, TS vs SS, with and
// without a concurrent tcgen05.ld stream from 4 other warps.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/probe_tslat tools/probe_ts_lat.cu
#include <cuda_runtime.h>
#include <cstdio>
#include "../paper_2404_03617_b200/csrc/sm100.cuh"
#include "../paper_2404_03617_b200/csrc/common.cuh"
using namespace wl;

template <int N, int MODE, int LD>
__global__ void k_lat(long long* out, int reps) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tb;
  __shared__ volatile int stop;
  for (int i = threadIdx.x; i < 160 * 1024 / 16; i += blockDim.x) reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  if (threadIdx.x < 32) tmem_alloc<512>(&tb);
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    stop = 0;
    fence_mbar_init();
  }
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tb;
  const int warp = threadIdx.x / 32;
  if (threadIdx.x == 0) {
    const uint32_t idesc = make_idesc_f16(128, N);
    const uint32_t a0 = smem_u32(smem), b0 = smem_u32(smem + 65536);
    long long tot = 0;
    for (int r = 0; r < reps; ++r) {
      long long t0 = clock64();
      for (int t = 0; t < 2; ++t)
        for (int k = 0; k < 8; ++k) {
          const uint32_t d = tmem + 256 + t * N;
          const uint64_t bd = make_sdesc(b0 + k * 2 * N * 16, N * 16, 128);
          if (MODE == 0) mma_ss(d, make_sdesc(a0 + t * 2048 + k * 2 * 4096, 4096, 128), bd, idesc, k > 0);
          else mma_ts(d, tmem + t * 64 + k * 8, bd, idesc, k > 0);
        }
      mma_commit(&bar);
      mbar_wait(&bar, r & 1);
      tot += clock64() - t0;
    }
    out[0] = tot / reps;
    stop = 1;
  } else if (LD == 1 && warp >= 4 && warp < 8) {
    const int q = warp % 4;
    uint32_t acc = 0;
    while (!stop) {
      uint32_t v[16];
      WL_TMEM_LD16(tmem_lane_addr(tmem, q, 384), v);
      tmem_ld_wait();
      acc += v[0];
    }
    if (acc == 12345) out[1] = acc;
  } else if (LD == 2 && warp >= 4 && warp < 8) {
    // the FFN epilogue's pattern: tcgen05.ld 16 columns + tcgen05.st 8 packed columns
    const int q = warp % 4;
    uint32_t acc = 0;
    while (!stop) {
      uint32_t v[16];
      WL_TMEM_LD16(tmem_lane_addr(tmem, q, 384), v);
      tmem_ld_wait();
      uint32_t o[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) o[i] = v[2 * i] ^ v[2 * i + 1];
      WL_TMEM_ST8(tmem_lane_addr(tmem, q, 448), o);
      tmem_st_wait();
      acc += v[0];
    }
    if (acc == 12345) out[1] = acc;
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc<512>(tmem);
}

template <int N, int MODE, int LD>
void run() {
  long long* d;
  cudaMalloc(&d, 16);
  auto k = k_lat<N, MODE, LD>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 164 * 1024);
  k<<<1, 256, 164 * 1024>>>(d, 4);
  k<<<1, 256, 164 * 1024>>>(d, 200);
  long long h;
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("%s N=%3d tcgen05.ld load %d: 16 MMAs + commit = %lld cycles  %s\n", MODE ? "TS" : "SS", N, LD, h,
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

int main() {
  run<64, 0, 0>();
  run<64, 1, 0>();
  run<64, 0, 1>();
  run<64, 1, 1>();
  run<128, 1, 0>();
  run<128, 1, 1>();
  run<64, 0, 2>();
  run<64, 1, 2>();
  run<128, 1, 2>();
  return 0;
}
