// probe_hmma.cu — legacy warp-level mma.sync throughput on sm_100a (the
// paper's m16n8k8 instruction, K = 8 = T, no block-diagonal waste) and
// whether it overlaps tcgen05.mma issued by another warp of the same CTA.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/probe_hmma tools/probe_hmma.cu
#include <cuda_runtime.h>
#include <cstdio>
#include "../paper_2404_03617_b200/csrc/sm100.cuh"
using namespace wl;

// SHAPE 0: m16n8k8 f32 acc; 1: m16n8k16 f32 acc; 2: m16n8k16 f16 acc; 3: m16n8k8 f16 acc
template <int SHAPE, int ILP>
__device__ __forceinline__ void hmma_loop(int iters, uint32_t a0, uint32_t a1, uint32_t b0, float* sink) {
  float acc[ILP][4];
  uint32_t hacc[ILP][2];
#pragma unroll
  for (int i = 0; i < ILP; ++i) {
    acc[i][0] = acc[i][1] = acc[i][2] = acc[i][3] = 0.f;
    hacc[i][0] = hacc[i][1] = 0;
  }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i) {
      if (SHAPE == 0) {
        asm volatile(
            "mma.sync.aligned.m16n8k8.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
            : "+f"(acc[i][0]), "+f"(acc[i][1]), "+f"(acc[i][2]), "+f"(acc[i][3])
            : "r"(a0), "r"(a1), "r"(b0));
      } else if (SHAPE == 1) {
        asm volatile(
            "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
            "{%0,%1,%2,%3};"
            : "+f"(acc[i][0]), "+f"(acc[i][1]), "+f"(acc[i][2]), "+f"(acc[i][3])
            : "r"(a0), "r"(a1), "r"(a0), "r"(a1), "r"(b0), "r"(b0));
      } else if (SHAPE == 2) {
        asm volatile(
            "mma.sync.aligned.m16n8k16.row.col.f16.f16.f16.f16 {%0,%1}, {%2,%3,%4,%5}, {%6,%7}, {%0,%1};"
            : "+r"(hacc[i][0]), "+r"(hacc[i][1])
            : "r"(a0), "r"(a1), "r"(a0), "r"(a1), "r"(b0), "r"(b0));
      } else {
        asm volatile("mma.sync.aligned.m16n8k8.row.col.f16.f16.f16.f16 {%0,%1}, {%2,%3}, {%4}, {%0,%1};"
                     : "+r"(hacc[i][0]), "+r"(hacc[i][1])
                     : "r"(a0), "r"(a1), "r"(b0));
      }
    }
  }
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < ILP; ++i) s += acc[i][0] + acc[i][1] + acc[i][2] + acc[i][3] + __uint_as_float(hacc[i][0]);
  if (s == 1234.5f) *sink = s;
}

// warps [0, hw) run mma.sync; if TC, warp hw (one thread) streams tcgen05 N=TCN MMAs
template <int SHAPE, int ILP, bool TC, int TCN>
__global__ void k_hmma(long long* out, int iters, int tc_iters, int hw, float* sink) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tb;
  const int wid = threadIdx.x / 32;
  if (TC) {
    for (int i = threadIdx.x; i < 96 * 1024 / 16; i += blockDim.x) reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
    if (wid == 0) tmem_alloc<512>(&tb);
    if (threadIdx.x == 0) {
      mbar_init(&bar, 1);
      fence_mbar_init();
    }
    fence_async_smem();
    tc_fence_before();
  }
  __syncthreads();
  if (TC) tc_fence_after();
  long long t0 = clock64();
  if (wid < hw) {
    const uint32_t a0 = 0x3c003c00u ^ threadIdx.x, a1 = 0x3c003c00u, b0 = 0x3c003c00u;
    hmma_loop<SHAPE, ILP>(iters, a0, a1, b0, sink);
    __syncwarp();
    if (threadIdx.x % 32 == 0) out[1 + wid] = clock64() - t0;
  } else if (TC && wid == hw && threadIdx.x % 32 == 0) {
    const uint32_t tmem = tb;
    const uint32_t idesc = make_idesc_f16(128, TCN);
    const uint32_t sa = smem_u32(smem), sb = smem_u32(smem + 65536);
    uint64_t ad[8], bd[8];
    for (int i = 0; i < 8; ++i) {
      ad[i] = make_sdesc(sa + i * 256, 2048, 128);
      bd[i] = make_sdesc(sb + i * 256, TCN * 16, 128);
    }
    for (int it = 0; it < tc_iters; ++it) {
#pragma unroll
      for (int k = 0; k < 8; ++k) mma_ss(tmem + (k & 1) * 256, ad[k], bd[k], idesc, 1);
    }
    mma_commit(&bar);
    mbar_wait(&bar, 0);
    out[0] = clock64() - t0;
  }
  if (TC) {
    tc_fence_before();
    __syncthreads();
    if (wid == 0) tmem_dealloc<512>(tb);
  }
}

static const char* shape_name(int s) {
  switch (s) {
    case 0: return "m16n8k8  f32acc";
    case 1: return "m16n8k16 f32acc";
    case 2: return "m16n8k16 f16acc";
    default: return "m16n8k8  f16acc";
  }
}
static int shape_macs(int s) { return (s == 0 || s == 3) ? 16 * 8 * 8 : 16 * 8 * 16; }

template <int SHAPE, int ILP, bool TC, int TCN = 128>
void run(int hw, int tc_iters = 0) {
  long long* d;
  float* sink;
  cudaMalloc(&d, 8 * 64);
  cudaMalloc(&sink, 4);
  cudaMemset(d, 0, 8 * 64);
  auto k = k_hmma<SHAPE, ILP, TC, TCN>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  const int iters = 4000;
  const int threads = 32 * (hw + (TC ? 1 : 0));
  k<<<1, threads, 100 * 1024>>>(d, 10, TC ? 2 : 0, hw, sink);
  k<<<1, threads, 100 * 1024>>>(d, iters, tc_iters, hw, sink);
  long long h[64];
  cudaMemcpy(h, d, 8 * 64, cudaMemcpyDeviceToHost);
  long long mx = 0;
  for (int w = 0; w < hw; ++w) mx = h[1 + w] > mx ? h[1 + w] : mx;
  const double macs = (double)hw * iters * ILP * shape_macs(SHAPE);
  printf("%s warps=%2d ILP=%d  %7.1f MAC/cycle/SM (%.2f cyc per mma per warp)", shape_name(SHAPE), hw, ILP,
         macs / mx, (double)mx / (iters * ILP));
  if (TC) {
    const double tcmacs = (double)tc_iters * 8 * 128 * TCN * 16;
    printf("  | tcgen05 N=%d alone-equiv: %.1f MAC/cycle over %lld cyc", TCN, tcmacs / h[0], h[0]);
  }
  printf("  %s\n", cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
  cudaFree(sink);
}

// two CTAs on one SM each issuing N=16 tcgen05 MMAs: is the ~44-cycle floor per CTA or per SM?
template <int N>
__global__ void k_tc2(long long* out, int iters) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tb;
  for (int i = threadIdx.x; i < 80 * 1024 / 16; i += blockDim.x) reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  if (threadIdx.x < 32) tmem_alloc<128>(&tb);
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
    const uint32_t idesc = make_idesc_f16(128, N);
    const uint32_t a0 = smem_u32(smem), b0 = smem_u32(smem + 65536);
    uint64_t ad[8], bd[8];
    for (int i = 0; i < 8; ++i) {
      ad[i] = make_sdesc(a0 + i * 256, 2048, 128);
      bd[i] = make_sdesc(b0 + i * 256, N * 16, 128);
    }
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int k = 0; k < 8; ++k) mma_ss(tmem + (k & 3) * 32, ad[k], bd[k], idesc, 1);
    }
    mma_commit(&bar);
    mbar_wait(&bar, 0);
    out[2 * blockIdx.x] = clock64() - t0;
    out[2 * blockIdx.x + 1] = smid;
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc<128>(tmem);
}

template <int N>
void run_tc2(int ctas) {
  long long* d;
  cudaMalloc(&d, 8 * 2 * 512);
  auto k = k_tc2<N>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 82 * 1024);
  const int iters = 2000;
  k<<<ctas, 128, 82 * 1024>>>(d, 10);
  k<<<ctas, 128, 82 * 1024>>>(d, iters);
  long long h[2 * 512];
  cudaMemcpy(h, d, 8 * 2 * ctas, cudaMemcpyDeviceToHost);
  // CTAs sharing SM 0's id
  int n_same = 0;
  long long mx = 0;
  for (int c = 0; c < ctas; ++c)
    if (h[2 * c + 1] == h[1]) {
      ++n_same;
      mx = h[2 * c] > mx ? h[2 * c] : mx;
    }
  printf("tcgen05 N=%d, %d CTAs (%d on SM %lld): %.2f cycles per MMA per CTA  %s\n", N, ctas, n_same, h[1],
         (double)mx / (iters * 8), cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

int main() {
  // legacy HMMA peak per SM
  for (int hw : {4, 8, 16}) {
    run<0, 4, false>(hw);
    run<0, 8, false>(hw);
  }
  for (int hw : {4, 8, 16}) run<1, 4, false>(hw);
  for (int hw : {4, 8, 16}) run<2, 4, false>(hw);
  for (int hw : {4, 8}) run<3, 4, false>(hw);
  // overlap with tcgen05 (one issuing warp) — N=128 (dense) and N=16 (conv-like)
  run<0, 4, true, 128>(8, 300);
  run<0, 4, true, 128>(0, 300);
  run<0, 4, true, 16>(8, 300);
  run<0, 4, true, 16>(0, 300);
  run<1, 4, true, 128>(8, 300);
  // two CTAs per SM (2 x 82 KB smem) each issuing N=16 / N=64 / N=128
  run_tc2<16>(148);
  run_tc2<16>(296);
  run_tc2<64>(148);
  run_tc2<64>(296);
  run_tc2<128>(148);
  run_tc2<128>(296);
  return 0;
}
