// gemm.cu — persistent tcgen05 GEMM with a fused epilogue for the pointwise
// contractions that are not inside a fused block: the layer-wise FFN schedule
// (machine.py:339-365: X U + a -> phi -> . V + b, hidden through memory), and
// the ConvNeXt-T units that have no fused form in the paper (patchify stem,
// LayerNorm + 2x2 stride-2 downsample, the C = 768 stage's expand / project
// with the hidden L2-resident, the classifier).
//
// Tile 128 x BN (BN <= 256) x 64: A and B arrive by TMA in the 128-byte
// swizzled K-major layout (one box each per K step), a ring of up to 8 stages;
// one thread issues 4 x tcgen05.mma (K = 16) per stage into one of two TMEM
// accumulators, so the epilogue of tile i overlaps the main loop of tile i+1.
// Warps: 0 TMA producer, 1 MMA issuer, 2-5 epilogue (TMEM lane quadrant =
// warp % 4; thread = output row). Grid = min(tiles, SMs), tiles strided.
#include <cuda.h>
#include <cuda_fp16.h>
#include <cstdint>
#include <cstring>
#include "common.cuh"
#include "gemm.h"
#include "launch.h"
#include "plan.h"

namespace wl {

namespace gm {
constexpr int kThreads = 192;
constexpr int kBK = 64;
constexpr int kMaxStages = 8;
constexpr int kSmemMax = 232448;
struct Args {
  int M, N, BN, tiles_m, tiles, kblocks, stages, stage_bytes;
  int ldd, ldr, act;
  float ln_eps;
  const float* bias;
  const float* ln_g;
  const float* ln_b;
  const __half* res;
  __half* D;
  uint32_t tmem_cols;
};
struct Bars {
  uint64_t full[kMaxStages], empty[kMaxStages];
  uint64_t acc_full[2], acc_empty[2];
  uint32_t tmem_base;
};
}  // namespace gm

__device__ __forceinline__ void tma_load_2d(void* dst, const void* tmap, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
      "[%4];" ::"r"(smem_u32(dst)),
      "l"(tmap), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ float act_rt(float v, int a) {
  switch (a) {
    case kRelu: return act<kRelu>(v);
    case kSilu: return act<kSilu>(v);
    case kSigmoid: return act<kSigmoid>(v);
    case kGelu: return act<kGelu>(v);
  }
  return v;
}

// bias + activation of 16 accumulators at output column n (n + 16 may pass N)
__device__ __forceinline__ void gemm_pre(const gm::Args& a, const uint32_t* v, int n, float* f) {
#pragma unroll
  for (int i = 0; i < 16; ++i) f[i] = __uint_as_float(v[i]);
  if (a.bias) {
    if (n + 16 <= a.N) {
      float b[16];
      load16f(a.bias + n, b);
#pragma unroll
      for (int i = 0; i < 16; ++i) f[i] += b[i];
    } else {
#pragma unroll
      for (int i = 0; i < 16; ++i)
        if (n + i < a.N) f[i] += a.bias[n + i];
    }
  }
  if (a.act != kIdentity) {
#pragma unroll
    for (int i = 0; i < 16; ++i) f[i] = act_rt(f[i], a.act);
  }
}

__global__ void __launch_bounds__(gm::kThreads, 1)
    gemm_kernel(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tb,
                const __grid_constant__ gm::Args a) {
  using namespace gm;
  extern __shared__ __align__(1024) uint8_t smem[];
  Bars& B = *reinterpret_cast<Bars*>(smem + a.stages * a.stage_bytes);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < a.stages; ++s) {
      mbar_init(&B.full[s], 1);
      mbar_init(&B.empty[s], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&B.acc_full[i], 1);
      mbar_init(&B.acc_empty[i], 4);
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc_n(&B.tmem_base, a.tmem_cols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  pdl_trigger();
  pdl_wait();
  const uint32_t tmem = B.tmem_base;

  if (warp == 0) {
    if (lane == 0) {
      // ---------------------------------------------------------- producer
      prefetch_tmap(&ta);
      prefetch_tmap(&tb);
      int s = 0;
      uint32_t ph = 0;
      for (int tile = blockIdx.x; tile < a.tiles; tile += gridDim.x) {
        const int tn = tile / a.tiles_m, tm = tile % a.tiles_m;
        for (int kb = 0; kb < a.kblocks; ++kb) {
          mbar_wait(&B.empty[s], ph ^ 1);
          uint8_t* st = smem + s * a.stage_bytes;
          mbar_arrive_expect_tx(&B.full[s], a.stage_bytes);
          tma_load_2d(st, &ta, kb * kBK, tm * 128, &B.full[s]);
          tma_load_2d(st + 16384, &tb, kb * kBK, tn * a.BN, &B.full[s]);
          if (++s == a.stages) {
            s = 0;
            ph ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---------------------------------------------------------- MMA issuer
      const uint32_t idesc = make_idesc_f16(128, a.BN);
      int s = 0;
      uint32_t ph = 0;
      int it = 0;
      for (int tile = blockIdx.x; tile < a.tiles; tile += gridDim.x, ++it) {
        const int ab = it & 1, u = it >> 1;
        mbar_wait(&B.acc_empty[ab], (u & 1) ^ 1);
        tc_fence_after();
        const uint32_t d = tmem + ab * (a.tmem_cols / 2);
        for (int kb = 0; kb < a.kblocks; ++kb) {
          mbar_wait(&B.full[s], ph);
          tc_fence_after();
          const uint32_t sa = smem_u32(smem + s * a.stage_bytes), sb = sa + 16384;
#pragma unroll
          for (int k = 0; k < 4; ++k)
            mma_ss(d, make_sdesc_sw128(sa + k * 32), make_sdesc_sw128(sb + k * 32), idesc, (kb | k) != 0);
          mma_commit(&B.empty[s]);
          if (++s == a.stages) {
            s = 0;
            ph ^= 1;
          }
        }
        mma_commit(&B.acc_full[ab]);
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue
    const int q = warp & 3;
    int it = 0;
    for (int tile = blockIdx.x; tile < a.tiles; tile += gridDim.x, ++it) {
      const int ab = it & 1, u = it >> 1;
      const int tn = tile / a.tiles_m, tm = tile % a.tiles_m;
      mbar_wait(&B.acc_full[ab], u & 1);
      tc_fence_after();
      const int row = tm * 128 + q * 32 + lane;
      const uint32_t tb0 = tmem_lane_addr(tmem, q, ab * (a.tmem_cols / 2));
      const int n0 = tn * a.BN;
      float mean = 0.f, rstd = 1.f;
      if (a.ln_g) {
        // row LayerNorm over the whole output row (tiles_n == 1): two-pass
        // statistics from TMEM (mean, then centred second moment)
        float s1 = 0.f;
        for (int c0 = 0; c0 < a.BN; c0 += 16) {
          uint32_t v[16];
          WL_TMEM_LD16(tb0 + c0, v);
          tmem_ld_wait();
          float f[16];
          gemm_pre(a, v, n0 + c0, f);
#pragma unroll
          for (int i = 0; i < 16; ++i)
            if (n0 + c0 + i < a.N) s1 += f[i];
        }
        mean = s1 / (float)a.N;
        float s2 = 0.f;
        for (int c0 = 0; c0 < a.BN; c0 += 16) {
          uint32_t v[16];
          WL_TMEM_LD16(tb0 + c0, v);
          tmem_ld_wait();
          float f[16];
          gemm_pre(a, v, n0 + c0, f);
#pragma unroll
          for (int i = 0; i < 16; ++i)
            if (n0 + c0 + i < a.N) s2 += (f[i] - mean) * (f[i] - mean);
        }
        rstd = rsqrtf(s2 / (float)a.N + a.ln_eps);
      }
      for (int c0 = 0; c0 < a.BN; c0 += 16) {
        uint32_t v[16];
        WL_TMEM_LD16(tb0 + c0, v);
        tmem_ld_wait();
        const int n = n0 + c0;
        if (row < a.M && n < a.N) {
          float f[16];
          gemm_pre(a, v, n, f);
          if (a.ln_g) {
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              const int c = n + i < a.N ? n + i : a.N - 1;
              f[i] = (f[i] - mean) * rstd * a.ln_g[c] + a.ln_b[c];
            }
          }
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            if (n + 8 * h >= a.N) break;
            float* g = f + 8 * h;
            if (a.res) {
              float r[8];
              unpack8(__ldg(reinterpret_cast<const uint4*>(a.res + (size_t)row * a.ldr + n + 8 * h)), r);
#pragma unroll
              for (int i = 0; i < 8; ++i) g[i] += r[i];
            }
            *reinterpret_cast<uint4*>(a.D + (size_t)row * a.ldd + n + 8 * h) = pack8(g);
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&B.acc_empty[ab]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    __syncwarp();
    tmem_dealloc_n(tmem, a.tmem_cols);
  }
}

// =================================================================== host
static int pick_bn(int N) {
  if (N <= 256) return align_up(N, 16);
  int best = 256, waste = 1 << 30;
  for (int bn : {256, 192, 128}) {
    const int w = ((N + bn - 1) / bn) * bn - N;
    if (w < waste) {
      waste = w;
      best = bn;
    }
  }
  return best;
}

int gemm_run(const void* A, int M, int K, int lda, const void* Bw, int N, int ldb, void* D, int ldd,
             const GemmEpi& e, cudaStream_t st) {
  if (M < 1 || N < 1 || K < 1 || K % 8 || lda % 8 || ldb % 8 || ldd % 8 || N % 8 || (e.res && e.ldr % 8))
    return set_error(WL_EINVAL, "gemm: M=%d N=%d K=%d lda=%d ldb=%d ldd=%d: sizes/strides must be multiples of 8", M,
                     N, K, lda, ldb, ldd);
  gm::Args a;
  memset(&a, 0, sizeof(a));
  a.M = M;
  a.N = N;
  a.BN = pick_bn(N);
  if (e.ln_g && a.BN < N) return set_error(WL_EUNSUPPORTED, "gemm: row LayerNorm needs N <= 256 (N = %d)", N);
  a.tiles_m = (M + 127) / 128;
  a.tiles = a.tiles_m * ((N + a.BN - 1) / a.BN);
  a.kblocks = (K + gm::kBK - 1) / gm::kBK;
  a.stage_bytes = 16384 + a.BN * 128;
  a.stages = (gm::kSmemMax - (int)sizeof(gm::Bars) - 64) / a.stage_bytes;
  if (a.stages > gm::kMaxStages) a.stages = gm::kMaxStages;
  a.ldd = ldd;
  a.ldr = e.ldr;
  a.act = e.act;
  a.ln_eps = e.ln_eps;
  a.bias = e.bias;
  a.ln_g = e.ln_g;
  a.ln_b = e.ln_b;
  a.res = e.res;
  a.D = reinterpret_cast<__half*>(D);
  a.tmem_cols = 32;
  while (a.tmem_cols < (uint32_t)(2 * a.BN)) a.tmem_cols *= 2;
  CUtensorMap tA, tB;
  {
    const uint64_t dims[2] = {(uint64_t)K, (uint64_t)M};
    const uint64_t strides[1] = {(uint64_t)lda * 2};
    const uint32_t box[2] = {64, 128};
    if (int r = encode_tmap(&tA, A, 2, dims, strides, box, true)) return r;
  }
  {
    const uint64_t dims[2] = {(uint64_t)K, (uint64_t)N};
    const uint64_t strides[1] = {(uint64_t)ldb * 2};
    const uint32_t box[2] = {64, (uint32_t)a.BN};
    if (int r = encode_tmap(&tB, Bw, 2, dims, strides, box, true)) return r;
  }
  const int smem = a.stages * a.stage_bytes + (int)sizeof(gm::Bars);
  const int grid = a.tiles < kNumSMs ? a.tiles : kNumSMs;
  return launch_pdl(gemm_kernel, grid, gm::kThreads, smem, st, "gemm launch", tA, tB, a);
}

int gemm_init() {
  return check_cuda(cudaFuncSetAttribute(gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, gm::kSmemMax),
                    "cudaFuncSetAttribute(gemm)");
}

}  // namespace wl
