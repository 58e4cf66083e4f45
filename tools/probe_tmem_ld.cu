// probe_tmem_ld.cu — tcgen05.ld throughput: cycles for 4 (or 8) warps to read
// NCOL fp32 columns of all 128 lanes, batched 4 x16 loads per wait, with and
// without concurrent MMAs (N=16 SS, one issuing thread) on other TMEM columns.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o probe_tmem tools/probe_tmem_ld.cu
#include <cuda_runtime.h>
#include <cstdio>
#include "../paper_2404_03617_b200/csrc/sm100.cuh"
using namespace wl;

template <int NCOL, int WARPS, bool MMA, int SHAPE>
__global__ void k_ld(long long* out, float* sink) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tb;
  __shared__ uint64_t bar;
  for (int i = threadIdx.x; i < 64 * 1024 / 16; i += blockDim.x) reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  if (threadIdx.x < 32) tmem_alloc<512>(&tb);
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tb;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  long long t0 = clock64();
  if (warp < WARPS) {
    const int q = warp % 4, half = warp / 4;
    float acc = 0.f;
    for (int rep = 0; rep < 16; ++rep) {
      for (int c = half * 16; c < NCOL; c += (WARPS / 4) * 16 * (SHAPE == 16 ? 1 : 2)) {
        uint32_t v[32];
        if (SHAPE == 16) {
          WL_TMEM_LD16(tmem + ((uint32_t)(q * 32) << 16) + c, v);
        } else {
          WL_TMEM_LD16(tmem + ((uint32_t)(q * 32) << 16) + c, v);
          uint32_t* v2 = v + 16;
          WL_TMEM_LD16(tmem + ((uint32_t)(q * 32) << 16) + c + 16, v2);
        }
        tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < (SHAPE == 16 ? 16 : 32); ++i) acc += __uint_as_float(v[i]);
      }
    }
    sink[threadIdx.x] = acc;
  } else if (MMA && warp == WARPS && lane == 0) {
    const uint32_t idesc = make_idesc_f16(128, 16);
    const uint64_t ad = make_sdesc(smem_u32(smem), 2048, 128), bd = make_sdesc(smem_u32(smem + 32768), 256, 128);
    for (int i = 0; i < 400; ++i) mma_ss(tmem + 384 + (i % 8) * 16, ad, bd, idesc, 1);
    mma_commit(&bar);
    mbar_wait(&bar, 0);
  }
  long long t1 = clock64();
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) out[0] = t1 - t0;
  if (threadIdx.x < 32) tmem_dealloc<512>(tmem);
}

template <int NCOL, int WARPS, bool MMA, int SHAPE>
void run() {
  long long* d; float* s;
  cudaMalloc(&d, 8); cudaMalloc(&s, 4096);
  auto k = k_ld<NCOL, WARPS, MMA, SHAPE>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  k<<<1, (WARPS + 1) * 32, 64 * 1024>>>(d, s);
  k<<<1, (WARPS + 1) * 32, 64 * 1024>>>(d, s);
  long long h;
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  const double bytes = 16.0 * NCOL * 128 * 4;
  printf("NCOL=%3d warps=%d mma=%d ld=x%d: %7.0f cycles for 16 passes -> %.1f B/cycle  %s\n", NCOL, WARPS, MMA, SHAPE, (double)h,
         bytes / h, cudaGetErrorString(cudaGetLastError()));
  cudaFree(d); cudaFree(s);
}

int main() {
  run<128, 4, false, 16>();
  run<128, 8, false, 16>();
  run<256, 4, false, 32>();
  run<256, 8, false, 32>();
  run<128, 4, true, 16>();
  run<128, 8, true, 16>();
  return 0;
}
