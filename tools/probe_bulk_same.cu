// probe_bulk_same.cu — L2 -> shared bulk-copy throughput when all 148 SMs read
// the SAME bytes at the same time (a weight stream shared by every CTA) vs
// distinct bytes, and with the reads of a shared stream multicast within
// clusters of 2 / 4 CTAs (one copy per cluster, delivered to every CTA).
#include <cuda_runtime.h>
#include <cstdio>
#include "../paper_2404_03617_b200/csrc/sm100.cuh"
using namespace wl;

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cl_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// MODE 0: distinct per SM; 1: same for all SMs; 2: same, multicast within the cluster (CS CTAs)
template <int MODE, int CS>
__global__ void k(const uint8_t* src, size_t src_bytes, long long* out, int iters, int chunk) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar[4], empty[4];
  constexpr int D = 4;
  const uint32_t rank = CS > 1 ? cluster_rank() : 0;
  if (threadIdx.x == 0) {
    for (int i = 0; i < D; ++i) {
      mbar_init(&bar[i], 1);
      mbar_init(&empty[i], CS);
    }
    fence_mbar_init();
  }
  __syncthreads();
  if (CS > 1) cl_sync();
  if (threadIdx.x == 0) {
    const size_t nchunk = src_bytes / chunk;
    long long t0 = clock64();
    for (int it = 0; it < iters + D; ++it) {
      const int b = it % D;
      if (it >= D) {
        mbar_wait(&bar[b], ((it / D) - 1) & 1);
        if (MODE == 2) {  // release the slot in every CTA of the cluster
          for (uint32_t c = 0; c < CS; ++c) {
            uint32_t ra;
            asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(smem_u32(&empty[b])), "r"(c));
            asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(ra) : "memory");
          }
        }
      }
      if (it < iters) {
        const size_t ci = MODE == 0 ? (blockIdx.x * 7919ull + it * 104729ull) % nchunk : (it * 104729ull) % nchunk;
        if (MODE == 2) {
          if (it >= D) mbar_wait(&empty[b], ((it / D) - 1) & 1);  // every CTA consumed the slot
          mbar_arrive_expect_tx(&bar[b], chunk);
          if ((uint32_t)(it % CS) == rank) {
            const uint16_t mask = (1u << CS) - 1;
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1], %2, "
                "[%3], %4;" ::"r"(smem_u32(smem + b * chunk)),
                "l"(src + ci * chunk), "r"(chunk), "r"(smem_u32(&bar[b])), "h"(mask)
                : "memory");
          }
        } else {
          mbar_arrive_expect_tx(&bar[b], chunk);
          bulk_g2s(smem + b * chunk, src + ci * chunk, chunk, &bar[b]);
        }
      }
    }
    out[blockIdx.x] = clock64() - t0;
  }
  __syncthreads();
  if (CS > 1) cl_sync();
}

template <int MODE, int CS>
void run(const uint8_t* src, size_t bytes, int chunk, const char* name) {
  long long* d;
  cudaMalloc(&d, 148 * 8);
  auto kk = k<MODE, CS>;
  cudaFuncSetAttribute(kk, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  const int iters = 64;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(148);
  cfg.blockDim = dim3(32);
  cfg.dynamicSmemBytes = 4 * chunk;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CS;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kk, src, bytes, d, 4, chunk);
  cudaLaunchKernelEx(&cfg, kk, src, bytes, d, iters, chunk);
  long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double mx = 0;
  for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
  printf("%-34s chunk %6d B, 4 in flight: %.1f B/cycle per SM delivered (all 148 SMs)  %s\n", name, chunk,
         (double)iters * chunk / mx, cudaGetErrorString(cudaGetLastError()));
}
int main() {
  const size_t bytes = 1u << 20;  // a 1 MB weight set, L2-resident
  uint8_t* src;
  cudaMalloc(&src, bytes);
  cudaMemset(src, 1, bytes);
  for (int chunk : {16384, 24576, 49152}) {
    run<0, 1>(src, bytes, chunk, "distinct bytes per SM");
    run<1, 1>(src, bytes, chunk, "same bytes on every SM");
    run<2, 2>(src, bytes, chunk, "same bytes, multicast x2 clusters");
    run<2, 4>(src, bytes, chunk, "same bytes, multicast x4 clusters");
  }
  return 0;
}
