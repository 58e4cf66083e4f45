// MUFU / FMA-pipe throughput of the activation building blocks on sm_100a:
// cycles per warp instruction per SM sub-partition, 8 independent chains per
// thread, `warps` warps per CTA, one CTA per SM.
#include <cstdio>
#include <cstdint>
#include <cuda_fp16.h>

template <int OP>
__device__ __forceinline__ uint32_t op(uint32_t x) {
  uint32_t r;
  if constexpr (OP == 0) asm volatile("tanh.approx.f16x2 %0, %1;" : "=r"(r) : "r"(x));
  if constexpr (OP == 1) asm volatile("tanh.approx.f32 %0, %1;" : "=r"(r) : "r"(x));
  if constexpr (OP == 2) asm volatile("ex2.approx.f16x2 %0, %1;" : "=r"(r) : "r"(x));
  if constexpr (OP == 3) asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=r"(r) : "r"(x));
  if constexpr (OP == 4) asm volatile("rcp.approx.ftz.f32 %0, %1;" : "=r"(r) : "r"(x));
  if constexpr (OP == 5) asm volatile("fma.rn.f16x2 %0, %1, %1, %1;" : "=r"(r) : "r"(x));
  if constexpr (OP == 6) asm volatile("tanh.approx.bf16x2 %0, %1;" : "=r"(r) : "r"(x));
  if constexpr (OP == 7) asm volatile("ex2.approx.ftz.bf16x2 %0, %1;" : "=r"(r) : "r"(x));
  return r;
}

template <int OP>
__global__ void probe(uint32_t* out, long long* cyc, int iters) {
  uint32_t v[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) v[k] = 0x3c003c00u + threadIdx.x + k;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = op<OP>(v[k]);
  }
  __syncthreads();
  long long t1 = clock64();
  uint32_t acc = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) acc ^= v[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int OP>
void run(const char* name, int warps) {
  uint32_t* out;
  long long* cyc;
  cudaMalloc(&out, 148 * 1024 * 4);
  cudaMalloc(&cyc, 148 * 8);
  const int iters = 256;
  probe<OP><<<148, warps * 32>>>(out, cyc, iters);
  probe<OP><<<148, warps * 32>>>(out, cyc, iters);
  cudaDeviceSynchronize();
  long long c;
  cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  // warp instructions per SM sub-partition = warps / 4 * iters * 8
  const double per = (double)c / ((double)warps / 4 * iters * 8);
  printf("%-22s warps %2d : %6.2f cycles per warp-instruction per SMSP\n", name, warps, per);
  cudaFree(out);
  cudaFree(cyc);
}

int main() {
  for (int w : {4, 8, 16}) {
    run<0>("tanh.approx.f16x2", w);
    run<1>("tanh.approx.f32", w);
    run<2>("ex2.approx.f16x2", w);
    run<3>("ex2.approx.f32", w);
    run<4>("rcp.approx.f32", w);
    run<5>("fma.rn.f16x2", w);
    run<6>("tanh.approx.bf16x2", w);
    run<7>("ex2.approx.bf16x2", w);
  }
  return 0;
}
