// probe_sw128.cu — validates SWIZZLE_128B K-major operands: TMA 2-D loads with
// 128-byte inner boxes + swizzle, UMMA descriptors with layout_type 2, K
// advance by +32 bytes inside the atom; also times 16-byte vs 128-byte boxes.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include "../paper_2404_03617_b200/csrc/sm100.cuh"
using namespace wl;
typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static PFN_encodeTiled enc;

__device__ __forceinline__ uint64_t sdesc_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;                  // LBO (unused for swizzled K-major)
  d |= (uint64_t)(1024 >> 4) << 32;        // SBO: 8 rows x 128 B
  d |= (uint64_t)1 << 46;                  // version
  d |= (uint64_t)2 << 61;                  // SWIZZLE_128B
  return d;
}

// D[128][N] = A[128][K] B[N][K]^T, K = 64 (one 128-byte swizzle atom per row)
template <int N>
__global__ void k_sw(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tb, float* D) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t bar, mbar;
  __shared__ uint32_t tb_;
  uint8_t* sA = smem;
  uint8_t* sB = smem + 16384;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (warp == 0) tmem_alloc<256>(&tb_);
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    mbar_init(&mbar, 1);
    fence_mbar_init();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tb_;
  if (threadIdx.x == 0) {
    mbar_arrive_expect_tx(&bar, 16384 + N * 128);
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                 ::"r"(smem_u32(sA)), "l"(&ta), "r"(0), "r"(0), "r"(smem_u32(&bar)) : "memory");
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                 ::"r"(smem_u32(sB)), "l"(&tb), "r"(0), "r"(0), "r"(smem_u32(&bar)) : "memory");
    mbar_wait(&bar, 0);
    tc_fence_after();
    const uint32_t idesc = make_idesc_f16(128, N);
    for (int kk = 0; kk < 4; ++kk)
      mma_ss(tmem, sdesc_sw128(smem_u32(sA)) + (uint64_t)(kk * 2), sdesc_sw128(smem_u32(sB)) + (uint64_t)(kk * 2),
             idesc, kk > 0);
    mma_commit(&mbar);
  }
  mbar_wait(&mbar, 0);
  tc_fence_after();
  const int row = warp * 32 + lane;
  for (int c0 = 0; c0 < N; c0 += 16) {
    uint32_t r[16];
    WL_TMEM_LD16(tmem + ((uint32_t)(warp * 32) << 16) + c0, r);
    tmem_ld_wait();
    for (int j = 0; j < 16; ++j) D[row * N + c0 + j] = __uint_as_float(r[j]);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<256>(tmem);
}

// TMA throughput: 16-byte-inner 3-D boxes vs 128-byte-inner swizzled 2-D boxes
__global__ void k_tma_rate(const __grid_constant__ CUtensorMap t16, const __grid_constant__ CUtensorMap t128,
                           int iters, long long* out, int rows) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t bar;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      mbar_arrive_expect_tx(&bar, 16384);
      asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                   ::"r"(smem_u32(smem)), "l"(&t16), "r"(0), "r"((i * 128) % rows), "r"(0), "r"(smem_u32(&bar)) : "memory");
      mbar_wait(&bar, i & 1);
    }
    long long t1 = clock64();
    for (int i = 0; i < iters; ++i) {
      mbar_arrive_expect_tx(&bar, 16384);
      asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                   ::"r"(smem_u32(smem)), "l"(&t128), "r"(0), "r"((i * 128) % rows), "r"(smem_u32(&bar)) : "memory");
      mbar_wait(&bar, (iters + i) & 1);
    }
    long long t2 = clock64();
    out[0] = t1 - t0;
    out[1] = t2 - t1;
  }
}

int main() {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  enc = (PFN_encodeTiled)fn;
  const int M = 128, N = 64, K = 64;
  std::vector<__half> hA(M * K), hB(N * K);
  std::vector<float> fA(M * K), fB(N * K);
  srand(7);
  for (int i = 0; i < M * K; ++i) { float v = (rand() % 17 - 8) / 8.f; hA[i] = __float2half(v); fA[i] = v; }
  for (int i = 0; i < N * K; ++i) { float v = (rand() % 17 - 8) / 8.f; hB[i] = __float2half(v); fB[i] = v; }
  __half *dA, *dB; float* dD;
  cudaMalloc(&dA, M * K * 2); cudaMalloc(&dB, N * K * 2); cudaMalloc(&dD, M * N * 4);
  cudaMemcpy(dA, hA.data(), M * K * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hB.data(), N * K * 2, cudaMemcpyHostToDevice);
  CUtensorMap ta, tb;
  cuuint64_t da[2] = {(cuuint64_t)K, (cuuint64_t)M}, sa[1] = {(cuuint64_t)K * 2};
  cuuint32_t ba[2] = {64, 128}, es[2] = {1, 1};
  enc(&ta, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, dA, da, sa, ba, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
      CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  cuuint64_t db[2] = {(cuuint64_t)K, (cuuint64_t)N};
  cuuint32_t bb[2] = {64, (cuuint32_t)N};
  enc(&tb, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, dB, db, sa, bb, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
      CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  cudaFuncSetAttribute(k_sw<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  k_sw<64><<<1, 128, 64 * 1024>>>(ta, tb, dD);
  cudaError_t e = cudaDeviceSynchronize();
  std::vector<float> D(M * N);
  cudaMemcpy(D.data(), dD, M * N * 4, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int m = 0; m < M; ++m)
    for (int n = 0; n < N; ++n) {
      double s = 0;
      for (int k = 0; k < K; ++k) s += (double)fA[m * K + k] * fB[n * K + k];
      if (fabs(s - D[m * N + n]) > 1e-3) { if (bad < 3) printf("  mismatch %d %d %f %f\n", m, n, D[m * N + n], s); ++bad; }
    }
  printf("SW128 K-major TMA+UMMA: %s bad=%d %s\n", cudaGetErrorString(e), bad, bad ? "FAIL" : "PASS");
  // TMA rate on a 64 MB buffer (rows of 512 halves)
  const int rows = 65536, cols = 512;
  __half* big;
  cudaMalloc(&big, (size_t)rows * cols * 2);
  cudaMemset(big, 0, (size_t)rows * cols * 2);
  CUtensorMap t16, t128;
  cuuint64_t d3[3] = {8, (cuuint64_t)rows, (cuuint64_t)(cols / 8)}, s3[2] = {(cuuint64_t)cols * 2, 16};
  cuuint32_t b3[3] = {8, 128, 8}, e3[3] = {1, 1, 1};
  enc(&t16, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 3, big, d3, s3, b3, e3, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
      CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  cuuint64_t d2[2] = {(cuuint64_t)cols, (cuuint64_t)rows}, s2[1] = {(cuuint64_t)cols * 2};
  cuuint32_t b2[2] = {64, 128};
  enc(&t128, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, big, d2, s2, b2, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
      CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  long long* dt;
  cudaMalloc(&dt, 16);
  cudaFuncSetAttribute(k_tma_rate, cudaFuncAttributeMaxDynamicSharedMemorySize, 40 * 1024);
  k_tma_rate<<<1, 32, 40 * 1024>>>(t16, t128, 64, dt, rows);
  k_tma_rate<<<1, 32, 40 * 1024>>>(t16, t128, 256, dt, rows);
  long long ht[2];
  cudaDeviceSynchronize();
  cudaMemcpy(ht, dt, 16, cudaMemcpyDeviceToHost);
  printf("TMA 16 KB tile, 1 SM, serial: 16-byte-inner 3-D box %.0f cycles, 128-byte swizzled 2-D box %.0f cycles (%s)\n",
         ht[0] / 256.0, ht[1] / 256.0, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
