// probe_sm100.cu — GPU microprobe validating the encodings in csrc/sm100.cuh:
// SS and TS tcgen05.mma with non-swizzled K-major layouts at arbitrary
// LBO/SBO, tcgen05.ld/st, 1-D bulk copy and 5-D TMA with OOB zero fill.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o probe tools/probe_sm100.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include "../paper_2404_03617_b200/csrc/sm100.cuh"

#define CK(x)                                                                      \
  do {                                                                             \
    cudaError_t e = (x);                                                           \
    if (e != cudaSuccess) {                                                        \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
      exit(1);                                                                     \
    }                                                                              \
  } while (0)

using namespace wl;

// D[M=128][N] = A[128][K] * B[N][K]^T ; A,B row-major fp16 (K contiguous)
template <int N, int K, bool TS>
__global__ void k_mma(const __half* A, const __half* B, float* D, int sboA, int lboA, int sboB, int lboB) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
  uint8_t* sA = smem;
  uint8_t* sB = smem + 64 * 1024;
  for (int i = tid; i < 128 * K; i += blockDim.x) {
    int r = i / K, k = i % K;
    *reinterpret_cast<__half*>(sA + (k / 8) * lboA + (r / 8) * sboA + (r % 8) * 16 + (k % 8) * 2) = A[i];
  }
  for (int i = tid; i < N * K; i += blockDim.x) {
    int r = i / K, k = i % K;
    *reinterpret_cast<__half*>(sB + (k / 8) * lboB + (r / 8) * sboB + (r % 8) * 16 + (k % 8) * 2) = B[i];
  }
  if (warp == 0) tmem_alloc<512>(&tbase);
  if (tid == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tbase;
  const uint32_t a_tmem = tmem + 256;  // columns 256.. hold A for the TS variant
  if (TS) {
    // lane = row, column j = (A[row][2j], A[row][2j+1]) packed
    const int row = (warp % 4) * 32 + lane;
    for (int c0 = 0; c0 < K / 2; c0 += 8) {
      uint32_t r[8];
      for (int j = 0; j < 8; ++j) {
        __half2 h = __halves2half2(A[row * K + 2 * (c0 + j)], A[row * K + 2 * (c0 + j) + 1]);
        r[j] = *reinterpret_cast<uint32_t*>(&h);
      }
      WL_TMEM_ST8(a_tmem + ((uint32_t)((warp % 4) * 32) << 16) + c0, r);
    }
    tmem_st_wait();
    tc_fence_before();
  }
  __syncthreads();
  tc_fence_after();
  if (tid == 0) {
    constexpr uint32_t idesc = make_idesc_f16(128, N);
    for (int kk = 0; kk < K / 16; ++kk) {
      uint64_t bd = make_sdesc(smem_u32(sB) + kk * 2 * lboB, lboB, sboB);
      if (TS) {
        mma_ts(tmem, a_tmem + kk * 8, bd, idesc, kk > 0);
      } else {
        uint64_t ad = make_sdesc(smem_u32(sA) + kk * 2 * lboA, lboA, sboA);
        mma_ss(tmem, ad, bd, idesc, kk > 0);
      }
    }
    mma_commit(&bar);
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  {
    const int row = (warp % 4) * 32 + lane;
    for (int c0 = 0; c0 < N; c0 += 16) {
      uint32_t r[16];
      WL_TMEM_LD16(tmem + ((uint32_t)((warp % 4) * 32) << 16) + c0, r);
      tmem_ld_wait();
      for (int j = 0; j < 16; ++j) D[row * N + c0 + j] = __uint_as_float(r[j]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tmem);
}

template <int N, int K, bool TS>
int run_mma(int sboA, int lboA, int sboB, int lboB) {
  std::vector<__half> hA(128 * K), hB(N * K);
  std::vector<float> fA(128 * K), fB(N * K), ref(128 * N), out(128 * N);
  srand(1234 + N + K);
  for (int i = 0; i < 128 * K; ++i) { float v = (rand() % 17 - 8) / 8.0f; hA[i] = __float2half(v); fA[i] = v; }
  for (int i = 0; i < N * K; ++i) { float v = (rand() % 17 - 8) / 8.0f; hB[i] = __float2half(v); fB[i] = v; }
  for (int m = 0; m < 128; ++m)
    for (int n = 0; n < N; ++n) {
      double s = 0;
      for (int k = 0; k < K; ++k) s += (double)fA[m * K + k] * fB[n * K + k];
      ref[m * N + n] = (float)s;
    }
  __half *dA, *dB; float* dD;
  CK(cudaMalloc(&dA, hA.size() * 2)); CK(cudaMalloc(&dB, hB.size() * 2)); CK(cudaMalloc(&dD, out.size() * 4));
  CK(cudaMemcpy(dA, hA.data(), hA.size() * 2, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, hB.data(), hB.size() * 2, cudaMemcpyHostToDevice));
  CK(cudaMemset(dD, 0, out.size() * 4));
  auto kern = k_mma<N, K, TS>;
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024));
  kern<<<1, 128, 160 * 1024>>>(dA, dB, dD, sboA, lboA, sboB, lboB);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(out.data(), dD, out.size() * 4, cudaMemcpyDeviceToHost));
  double maxerr = 0; int bad = 0;
  for (int i = 0; i < 128 * N; ++i) {
    double e = fabs(out[i] - ref[i]);
    if (e > maxerr) maxerr = e;
    if (e > 1e-3) { if (bad < 4) printf("   mismatch m=%d n=%d got %f ref %f\n", i / N, i % N, out[i], ref[i]); ++bad; }
  }
  printf("%s N=%d K=%d sboA=%d lboA=%d sboB=%d lboB=%d : maxerr %.3g bad %d -> %s\n", TS ? "TS" : "SS", N, K,
         sboA, lboA, sboB, lboB, maxerr, bad, bad ? "FAIL" : "PASS");
  cudaFree(dA); cudaFree(dB); cudaFree(dD);
  return bad ? 1 : 0;
}

// ---------------------------------------------------------------- TMA test
typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

// x: NHWC fp16 (N=2,H=6,W=7,C=32). View as 5-D (8ch, W, H, G, N) with the
// group stride 16 B so the box lands in smem as [G][Hb][Wb][8].
__global__ void k_tma(const __grid_constant__ CUtensorMap tmap, __half* out, int Wb, int Hb, int G, int n) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  __syncthreads();
  const uint32_t bytes = 8 * Wb * Hb * G * 2;
  if (threadIdx.x == 0) {
    mbar_arrive_expect_tx(&bar, bytes);
    tma_load_5d(smem, &tmap, 0, -1, -1, 0, n, &bar);
  }
  mbar_wait(&bar, 0);
  for (int i = threadIdx.x; i < (int)(bytes / 2); i += blockDim.x) out[i] = reinterpret_cast<__half*>(smem)[i];
}

__global__ void k_bulk(const uint4* src, uint4* dst, int n16) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    mbar_arrive_expect_tx(&bar, n16 * 16);
    bulk_g2s(smem, src, n16 * 16, &bar);
  }
  mbar_wait(&bar, 0);
  for (int i = threadIdx.x; i < n16; i += blockDim.x) dst[i] = reinterpret_cast<uint4*>(smem)[i];
}

int run_tma() {
  const int N = 2, H = 6, W = 7, C = 32, G = C / 8, Wb = W + 2, Hb = H + 2;
  std::vector<__half> hx(N * H * W * C);
  for (size_t i = 0; i < hx.size(); ++i) hx[i] = __float2half((float)(i % 2000) * 0.5f);
  __half *dx, *dout;
  CK(cudaMalloc(&dx, hx.size() * 2));
  CK(cudaMalloc(&dout, 8 * Wb * Hb * G * 2));
  CK(cudaMemcpy(dx, hx.data(), hx.size() * 2, cudaMemcpyHostToDevice));
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
  PFN_encodeTiled enc = (PFN_encodeTiled)fn;
  CUtensorMap tm;
  cuuint64_t dims[5] = {8, (cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)G, (cuuint64_t)N};
  cuuint64_t strides[4] = {(cuuint64_t)C * 2, (cuuint64_t)W * C * 2, 16, (cuuint64_t)H * W * C * 2};
  cuuint32_t box[5] = {8, (cuuint32_t)Wb, (cuuint32_t)Hb, (cuuint32_t)G, 1};
  cuuint32_t es[5] = {1, 1, 1, 1, 1};
  CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 5, dx, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) { printf("TMA encode failed %d -> FAIL\n", (int)r); return 1; }
  int bad = 0;
  for (int n = 0; n < N; ++n) {
    k_tma<<<1, 128, 8 * Wb * Hb * G * 2>>>(tm, dout, Wb, Hb, G, n);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    std::vector<__half> o(8 * Wb * Hb * G);
    CK(cudaMemcpy(o.data(), dout, o.size() * 2, cudaMemcpyDeviceToHost));
    for (int g = 0; g < G; ++g)
      for (int yy = 0; yy < Hb; ++yy)
        for (int xx = 0; xx < Wb; ++xx)
          for (int c = 0; c < 8; ++c) {
            int y = yy - 1, x = xx - 1;
            float e = (y < 0 || y >= H || x < 0 || x >= W) ? 0.f
                                                           : __half2float(hx[((n * H + y) * W + x) * C + g * 8 + c]);
            float got = __half2float(o[((g * Hb + yy) * Wb + xx) * 8 + c]);
            if (got != e) { if (bad < 4) printf("   tma mismatch n%d g%d y%d x%d c%d got %f exp %f\n", n, g, y, x, c, got, e); ++bad; }
          }
  }
  printf("TMA 5d halo load (G-stride 16B, negative coords): bad %d -> %s\n", bad, bad ? "FAIL" : "PASS");
  // bulk copy
  const int n16 = 1000;
  std::vector<uint4> hs(n16), ho(n16);
  for (int i = 0; i < n16; ++i) hs[i] = make_uint4(i, i * 3, i * 7, i ^ 0x55);
  uint4 *ds, *dd;
  CK(cudaMalloc(&ds, n16 * 16)); CK(cudaMalloc(&dd, n16 * 16));
  CK(cudaMemcpy(ds, hs.data(), n16 * 16, cudaMemcpyHostToDevice));
  k_bulk<<<1, 128, n16 * 16>>>(ds, dd, n16);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(ho.data(), dd, n16 * 16, cudaMemcpyDeviceToHost));
  int badb = 0;
  for (int i = 0; i < n16; ++i) badb += (ho[i].x != hs[i].x || ho[i].y != hs[i].y || ho[i].z != hs[i].z || ho[i].w != hs[i].w);
  printf("bulk copy 16000 B: bad %d -> %s\n", badb, badb ? "FAIL" : "PASS");
  return bad + badb ? 1 : 0;
}

int main() {
  int fails = 0;
  fails += run_mma<64, 64, false>(128, 128 * 16, 128, 64 * 16);      // dense
  fails += run_mma<16, 32, false>(144, 16 * 144 + 64, 160, 2 * 160 + 32);  // padded strides
  fails += run_mma<256, 64, false>(128, 2048, 128, 256 * 16);
  fails += run_mma<128, 32, false>(160, 2880, 128, 2048);          // conv-like strides
  fails += run_mma<64, 64, true>(128, 2048, 128, 64 * 16);         // A from TMEM
  fails += run_mma<128, 128, true>(128, 2048, 128, 128 * 16);
  fails += run_tma();
  printf(fails ? "PROBE FAIL (%d)\n" : "PROBE ALL PASS\n", fails);
  return fails ? 1 : 0;
}
