// probe_mma_contention.cu — cycles per M128 N16 K16 SS tcgen05.mma (one issuing
// thread) while other warps (a) idle, (b) stream LDS.128/STS.128 over shared
// memory, (c) stream tcgen05.ld from TMEM.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o probe_cont tools/probe_mma_contention.cu
#include <cuda_runtime.h>
#include <cstdio>
#include "../paper_2404_03617_b200/csrc/sm100.cuh"
using namespace wl;

template <int MODE, int NW, bool MMA = true>
__global__ void k(long long* out, float* sink, int iters) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tb;
  __shared__ volatile int done;
  for (int i = threadIdx.x; i < 160 * 1024 / 16; i += blockDim.x) reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  if (threadIdx.x < 32) tmem_alloc<512>(&tb);
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); done = 0; }
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tb;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0 && !MMA) {
    long long t0 = clock64();
    while (clock64() - t0 < 200000) {
    }
    out[0] = clock64() - t0;
    done = 1;
  } else if (threadIdx.x == 0) {
    const uint32_t idesc = make_idesc_f16(128, 16);
    const uint32_t a0 = smem_u32(smem), b0 = smem_u32(smem + 65536);
    uint64_t ad[8], bd[8];
    for (int i = 0; i < 8; ++i) { ad[i] = make_sdesc(a0 + i * 256, 4736, 128); bd[i] = make_sdesc(b0 + i * 256, 256, 128); }
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it)
#pragma unroll
      for (int j = 0; j < 8; ++j) mma_ss(tmem + (j % 4) * 16, ad[j], bd[j], idesc, 1);
    mma_commit(&bar);
    mbar_wait(&bar, 0);
    out[0] = clock64() - t0;
    done = 1;
  } else if (warp >= 4 && warp < 4 + NW) {
    float acc = 0.f;
    uint8_t* buf = smem + 98304 + (warp - 4) * 4096;
    const int q = warp % 4;
    long long nit = 0;
    while (!done) {
      ++nit;
      if (MODE == 1) {
        for (int r = 0; r < 16; ++r) {
          uint4 v = reinterpret_cast<uint4*>(buf)[(lane + r * 32) & 255];
          v.x += 1;
          reinterpret_cast<uint4*>(buf)[(lane * 7 + r * 32) & 255] = v;
        }
      } else if (MODE == 2) {
        uint32_t v[16];
        WL_TMEM_LD16(tmem + ((uint32_t)(q * 32) << 16) + 256 + (warp % 8) * 16, v);
        tmem_ld_wait();
        acc += __uint_as_float(v[0]);
      }
    }
    sink[threadIdx.x] = acc;
    if (lane == 0) reinterpret_cast<long long*>(sink + 1024)[warp] = nit;
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc<512>(tmem);
}

template <int MODE, int NW, bool MMA = true>
void run(const char* what) {
  long long* d; float* s;
  cudaMalloc(&d, 8); cudaMalloc(&s, 16384);
  auto kk = k<MODE, NW, MMA>;
  cudaFuncSetAttribute(kk, cudaFuncAttributeMaxDynamicSharedMemorySize, 164 * 1024);
  kk<<<1, 640, 164 * 1024>>>(d, s, 10);
  kk<<<1, 640, 164 * 1024>>>(d, s, 500);
  long long h; cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  long long nit[32];
  cudaMemcpy(nit, s + 1024, sizeof(nit), cudaMemcpyDeviceToHost);
  const double bytes = (double)nit[4] * 16 * 32 * 32;  // warp 4: 16 x (LDS.128 + STS.128) per iteration
  printf("%-40s %6.2f cycles/MMA | warp4 smem %.1f B/cycle  %s\n", what, (double)h / 4000, bytes / h,
         cudaGetErrorString(cudaGetLastError()));
}
int main() {
  run<1, 8, false>("no MMA, 8 warps LDS/STS.128");
  run<1, 8, true>("N16 SS MMA + 8 warps LDS/STS.128");
  run<1, 16, false>("no MMA, 16 warps LDS/STS.128");
  run<1, 16, true>("N16 SS MMA + 16 warps LDS/STS.128");
  return 0;
}
