// probe_bulk_l2.cu — L2 -> shared memory throughput per SM for 1-D bulk copies
// (cp.async.bulk) of 25 KB, with D copies in flight, all 148 SMs at once,
// source buffer L2-resident (32 MB, pre-touched).
#include <cuda_runtime.h>
#include <cstdio>
#include "../paper_2404_03617_b200/csrc/sm100.cuh"
using namespace wl;

template <int D, bool WRITE_FIRST = false>
__global__ void k(const uint8_t* src, size_t src_bytes, long long* out, int iters, int chunk) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar[8];
  if (threadIdx.x == 0) {
    for (int i = 0; i < D; ++i) mbar_init(&bar[i], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (WRITE_FIRST && threadIdx.x == 0) {
    // this SM bulk-stores its own chunks first (as the MBConv front writes h2), then reads them back
    for (int it = 0; it < iters; ++it) {
      const size_t nchunk = src_bytes / chunk;
      uint8_t* dst = const_cast<uint8_t*>(src) + ((blockIdx.x * 7919ull + it * 104729ull) % nchunk) * chunk;
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(smem)),
                   "r"(chunk) : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    asm volatile("fence.proxy.async.global;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const size_t nchunk = src_bytes / chunk;
    long long t0 = clock64();
    for (int it = 0; it < iters + D; ++it) {
      const int b = it % D;
      if (it >= D) mbar_wait(&bar[b], ((it / D) - 1) & 1);
      if (it < iters) {
        mbar_arrive_expect_tx(&bar[b], chunk);
        bulk_g2s(smem + b * chunk, src + ((blockIdx.x * 7919ull + it * 104729ull) % nchunk) * chunk, chunk, &bar[b]);
      }
    }
    out[blockIdx.x] = clock64() - t0;
  }
}

template <int D, bool WF = false>
void run(const uint8_t* src, size_t bytes, int chunk) {
  long long* d;
  cudaMalloc(&d, 148 * 8);
  auto kk = k<D, WF>;
  cudaFuncSetAttribute(kk, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  const int iters = 64;
  kk<<<148, 32, D * chunk>>>(src, bytes, d, 4, chunk);
  kk<<<148, 32, D * chunk>>>(src, bytes, d, iters, chunk);
  long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double mx = 0;
  for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
  printf("%s chunk %6d B, %d in flight: %.1f B/cycle per SM (all 148 SMs)  %s\n", WF ? "after own bulk stores" : "clean", chunk, D, (double)iters * chunk / mx,
         cudaGetErrorString(cudaGetLastError()));
}
int main() {
  const size_t bytes = 32u << 20;
  uint8_t* src;
  cudaMalloc(&src, bytes);
  cudaMemset(src, 1, bytes);
  run<4>(src, bytes, 25088);
  run<4, true>(src, bytes, 25088);
  run<2, true>(src, bytes, 25088);
  return 0;
}
