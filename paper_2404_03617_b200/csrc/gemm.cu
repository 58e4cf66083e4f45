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
// Warps: 0 TMA producer, 1 MMA issuer, 2-9 epilogue (TMEM lane quadrant =
// warp % 4, two warps per quadrant splitting the columns; thread = output
// row). The epilogue stages the fp16 tile in shared memory in the 128-byte
// swizzled layout (a residual tile arrives there by TMA first) and leaves by
// TMA stores, so HBM sees whole lines. Grid = min(tiles, SMs), tiles strided.
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
constexpr int kGroups = 4;                  // epilogue warp groups per TMEM lane quadrant
constexpr int kEpiThreads = kGroups * 128;
constexpr int kThreads = 64 + kEpiThreads;  // warp 0 TMA, warp 1 MMA, then the epilogue warps
constexpr int kBK = 64;
constexpr int kMaxStages = 8;
constexpr int kSmemMax = 232448;
struct Args {
  int M, N, BN, tiles_m, tiles_n, tiles, kblocks, stages, stage_bytes, s_stage, slabs;
  int act, has_res;
  float ln_eps;
  const float* bias;
  const float* ln_g;
  const float* ln_b;
  uint32_t tmem_cols;
};
struct Bars {
  uint64_t full[kMaxStages], empty[kMaxStages];
  uint64_t acc_full[2], acc_empty[2];
  uint64_t res_full;
  uint32_t tmem_base;
  float ln_red[2][kGroups][128];  // row LayerNorm: [sum | centred sum][column group][row]
  alignas(16) float bias[256];  // the tile's bias slice (0 past N or without bias)
};
}  // namespace gm

__device__ __forceinline__ void tma_load_2d(void* dst, const void* tmap, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
      "[%4];" ::"r"(smem_u32(dst)),
      "l"(tmap), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_store_2d(const void* tmap, const void* src, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(tmap),
               "r"(smem_u32(src)), "r"(c0), "r"(c1)
               : "memory");
}
__device__ __forceinline__ void bulk_commit_g() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0_g() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait0_g() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void gm_bar(int n) { asm volatile("bar.sync 1, %0;" ::"r"(n) : "memory"); }

__device__ __forceinline__ float act_rt(float v, int a) {
  switch (a) {
    case kRelu: return act<kRelu>(v);
    case kSilu: return act<kSilu>(v);
    case kSigmoid: return act<kSigmoid>(v);
    case kGelu: return act<kGelu>(v);
  }
  return v;
}
__device__ __forceinline__ __half2 act_rt_h2(__half2 v, int a) {
  switch (a) {
    case kRelu: return act_h2<kRelu>(v);
    case kSilu: return act_h2<kSilu>(v);
    case kSigmoid: return act_h2<kSigmoid>(v);
    case kGelu: return act_h2<kGelu>(v);
  }
  return v;
}

// accumulators + bias of 16 columns at column c of the tile (bias staged in shared memory)
__device__ __forceinline__ void gemm_bias(const float* s_bias, const uint32_t* v, int c, float* f) {
  float b[16];
  load16f(s_bias + c, b);
#pragma unroll
  for (int i = 0; i < 16; ++i) f[i] = __uint_as_float(v[i]) + b[i];
}

template <typename T>
__global__ void __launch_bounds__(gm::kThreads, 1)
    gemm_kernel(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tb,
                const __grid_constant__ CUtensorMap td, const __grid_constant__ CUtensorMap tr,
                const __grid_constant__ gm::Args a) {
  using namespace gm;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* s_st = smem + a.s_stage;  // output staging: slabs of [128 rows][64 cols] fp16, 128B-swizzled
  Bars& B = *reinterpret_cast<Bars*>(smem + a.s_stage + a.slabs * 16384);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < a.stages; ++s) {
      mbar_init(&B.full[s], 1);
      mbar_init(&B.empty[s], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&B.acc_full[i], 1);
      mbar_init(&B.acc_empty[i], kEpiThreads / 32);
    }
    mbar_init(&B.res_full, 1);
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
        const int tm = tile / a.tiles_n, tn = tile % a.tiles_n;  // m-major: the CTAs of one wave share A tiles through L2
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
    {  // warp-converged issue: one elected lane issues each MMA / commit
      // ---------------------------------------------------------- MMA issuer
      const uint32_t idesc = make_idesc_f16(128, a.BN) | Dt<T>::kIdescAB;
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
            mma_ss_w(d, make_sdesc_sw128(sa + k * 32), make_sdesc_sw128(sb + k * 32), idesc, (kb | k) != 0);
          mma_commit_w(&B.empty[s]);
          if (++s == a.stages) {
            s = 0;
            ph ^= 1;
          }
        }
        mma_commit_w(&B.acc_full[ab]);
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue
    // warp w: TMEM lane quadrant w % 4 (rows 32 q .. 32 q + 31), column half
    // (w - 2) / 4 of the tile's 16-column units
    const int q = warp & 3, half = (warp - 2) >> 2;  // half: the warp's column group
    const bool leader = threadIdx.x == 64;
    const int units = a.BN / 16;
    const int u_lo = half * units / kGroups, u_hi = (half + 1) * units / kGroups;
    const int r = q * 32 + lane;  // row in the tile
    int it = 0;
    for (int tile = blockIdx.x; tile < a.tiles; tile += gridDim.x, ++it) {
      const int ab = it & 1, u = it >> 1;
      const int tm = tile / a.tiles_n, tn = tile % a.tiles_n;  // m-major: the CTAs of one wave share A tiles through L2
      const int n0 = tn * a.BN;
      if (leader) {
        bulk_wait_read0_g();  // the previous tile's stores have left the staging buffer
        if (a.has_res) {
          mbar_arrive_expect_tx(&B.res_full, a.slabs * 16384);
          for (int sl = 0; sl < a.slabs; ++sl) tma_load_2d(s_st + sl * 16384, &tr, n0 + sl * 64, tm * 128, &B.res_full);
        }
      }
      for (int c = threadIdx.x - 64; c < a.BN; c += kEpiThreads)
        B.bias[c] = (a.bias && n0 + c < a.N) ? a.bias[n0 + c] : 0.f;
      gm_bar(kEpiThreads);
      mbar_wait(&B.acc_full[ab], u & 1);
      tc_fence_after();
      const uint32_t tb0 = tmem_lane_addr(tmem, q, ab * (a.tmem_cols / 2));
      // stage one 16-column unit (fp16, 128B-swizzled; + residual from the staging tile)
      auto stage_unit = [&](int uu, uint4* o) {
        const int c16 = uu * 16, sl = c16 >> 6, c8 = (c16 & 63) >> 3;
        uint8_t* rowp = s_st + sl * 16384 + r * 128;
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          uint8_t* p = rowp + (((c8 + hh) ^ (r & 7)) << 4);
          if (a.has_res) {
            float rr[8], g[8];
            unpack8t<T>(lds128(p), rr);
            unpack8t<T>(o[hh], g);
#pragma unroll
            for (int i = 0; i < 8; ++i) g[i] += rr[i];
            o[hh] = pack8t<T>(g);
          }
          *reinterpret_cast<uint4*>(p) = o[hh];
        }
      };
      if (a.has_res) mbar_wait(&B.res_full, it & 1);
      if (a.ln_g) {
        // row LayerNorm over the whole output row (tiles_n == 1, N <= 128):
        // each warp keeps its part of the row (<= 2 units) in registers; the
        // groups' partial sums meet in shared memory (fixed order: deterministic);
        // two-pass statistics (mean, then the centred second moment), fp32
        uint32_t v[32];
#pragma unroll
        for (int j = 0; j < 2; ++j)
          if (u_lo + j < u_hi) WL_TMEM_LD16(tb0 + (u_lo + j) * 16, (v + 16 * j));
        tmem_ld_wait();
        float s1 = 0.f;
#pragma unroll
        for (int j = 0; j < 2; ++j)
          if (u_lo + j < u_hi) {
            float f[16];
            gemm_bias(B.bias, v + 16 * j, (u_lo + j) * 16, f);
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              v[16 * j + i] = __float_as_uint(f[i]);
              if (n0 + (u_lo + j) * 16 + i < a.N) s1 += f[i];
            }
          }
        B.ln_red[0][half][r] = s1;
        gm_bar(kEpiThreads);
        float mean = 0.f;
#pragma unroll
        for (int gq = 0; gq < kGroups; ++gq) mean += B.ln_red[0][gq][r];
        mean /= (float)a.N;
        float s2 = 0.f;
#pragma unroll
        for (int j = 0; j < 2; ++j)
          if (u_lo + j < u_hi)
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              const float d = __uint_as_float(v[16 * j + i]) - mean;
              if (n0 + (u_lo + j) * 16 + i < a.N) s2 += d * d;
            }
        B.ln_red[1][half][r] = s2;
        gm_bar(kEpiThreads);
        float var = 0.f;
#pragma unroll
        for (int gq = 0; gq < kGroups; ++gq) var += B.ln_red[1][gq][r];
        const float rstd = rsqrtf(var / (float)a.N + a.ln_eps);
#pragma unroll
        for (int j = 0; j < 2; ++j)
          if (u_lo + j < u_hi) {
            float f[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              const int n = n0 + (u_lo + j) * 16 + i, c = n < a.N ? n : a.N - 1;
              f[i] = (__uint_as_float(v[16 * j + i]) - mean) * rstd * __ldg(a.ln_g + c) + __ldg(a.ln_b + c);
            }
            uint4 o[2] = {pack8t<T>(f), pack8t<T>(f + 8)};
            stage_unit(u_lo + j, o);
          }
      } else {
        // 32 columns (two x16 TMEM loads) per wait
        for (int u0 = u_lo; u0 < u_hi; u0 += 2) {
          uint32_t v[32];
#pragma unroll
          for (int j = 0; j < 2; ++j)
            if (u0 + j < u_hi) WL_TMEM_LD16(tb0 + (u0 + j) * 16, (v + 16 * j));
          tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 2; ++j)
            if (u0 + j < u_hi) {
              float f[16];
              gemm_bias(B.bias, v + 16 * j, (u0 + j) * 16, f);
              uint4 o[2];
              uint32_t* ow = reinterpret_cast<uint32_t*>(o);
#pragma unroll
              for (int i = 0; i < 8; ++i) {
                if constexpr (Dt<T>::kIdescAB == 0) {
                  __half2 h = __floats2half2_rn(f[2 * i], f[2 * i + 1]);
                  if (a.act) h = act_rt_h2(h, a.act);
                  ow[i] = *reinterpret_cast<uint32_t*>(&h);
                } else {
                  ow[i] = Dt<T>::pack2(act_rt(f[2 * i], a.act), act_rt(f[2 * i + 1], a.act));
                }
              }
              stage_unit(u0 + j, o);
            }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&B.acc_empty[ab]);
      fence_async_smem();
      gm_bar(kEpiThreads);
      if (leader) {
        for (int sl = 0; sl < a.slabs; ++sl) tma_store_2d(&td, s_st + sl * 16384, n0 + sl * 64, tm * 128);
        bulk_commit_g();
      }
    }
    if (leader) bulk_wait0_g();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    __syncwarp();
    tmem_dealloc_n(tmem, a.tmem_cols);
  }
}

// =================================================================== host
static int pick_bn(int N, int tiles_m, bool whole_rows) {
  // few row tiles (e.g. the classifier, M = batch): 64-column tiles spread the
  // output over more SMs — each CTA's time is its A stream, not its N width
  // (not with the row-LayerNorm epilogue, which needs whole rows in one tile)
  if (!whole_rows && tiles_m * ((N + 255) / 256) < kNumSMs / 2) return N <= 64 ? align_up(N, 16) : 64;
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
             const GemmEpi& e, cudaStream_t st, int dtype) {
  if (M < 1 || N < 1 || K < 1 || K % 8 || lda % 8 || ldb % 8 || ldd % 8 || N % 8 || (e.res && e.ldr % 8))
    return set_error(WL_EINVAL, "gemm: M=%d N=%d K=%d lda=%d ldb=%d ldd=%d: sizes/strides must be multiples of 8", M,
                     N, K, lda, ldb, ldd);
  gm::Args a;
  memset(&a, 0, sizeof(a));
  a.M = M;
  a.N = N;
  a.BN = pick_bn(N, (M + 127) / 128, e.ln_g != nullptr);
  if (e.ln_g && (a.BN < N || N > 128 || e.act))
    return set_error(WL_EUNSUPPORTED, "gemm: the row-LayerNorm epilogue needs N <= 128 and no activation (N = %d)", N);
  a.tiles_m = (M + 127) / 128;
  a.tiles_n = (N + a.BN - 1) / a.BN;
  a.tiles = a.tiles_m * a.tiles_n;
  a.kblocks = (K + gm::kBK - 1) / gm::kBK;
  a.stage_bytes = 16384 + a.BN * 128;
  a.slabs = (a.BN + 63) / 64;
  a.stages = (gm::kSmemMax - a.slabs * 16384 - (int)sizeof(gm::Bars) - 64) / a.stage_bytes;
  if (a.stages > gm::kMaxStages) a.stages = gm::kMaxStages;
  a.s_stage = a.stages * a.stage_bytes;
  a.act = e.act;
  a.has_res = e.res != nullptr;
  a.ln_eps = e.ln_eps;
  a.bias = e.bias;
  a.ln_g = e.ln_g;
  a.ln_b = e.ln_b;
  a.tmem_cols = 32;
  while (a.tmem_cols < (uint32_t)(2 * a.BN)) a.tmem_cols *= 2;
  CUtensorMap tA, tB, tD, tR;
  auto map2 = [](CUtensorMap* m, const void* base, int inner, int outer, int ld, int box_outer) {
    const uint64_t dims[2] = {(uint64_t)inner, (uint64_t)outer};
    const uint64_t strides[1] = {(uint64_t)ld * 2};
    const uint32_t box[2] = {64, (uint32_t)box_outer};
    return encode_tmap(m, base, 2, dims, strides, box, true);
  };
  if (int r = map2(&tA, A, K, M, lda, 128)) return r;
  if (int r = map2(&tB, Bw, K, N, ldb, a.BN)) return r;
  if (int r = map2(&tD, D, N, M, ldd, 128)) return r;
  if (int r = map2(&tR, e.res ? (const void*)e.res : D, N, M, e.res ? e.ldr : ldd, 128)) return r;
  const int smem = a.s_stage + a.slabs * 16384 + (int)sizeof(gm::Bars);
  const int grid = a.tiles < kNumSMs ? a.tiles : kNumSMs;
  if (dtype == WL_DTYPE_BF16)
    return launch_pdl(gemm_kernel<__nv_bfloat16>, grid, gm::kThreads, smem, st, "gemm launch", tA, tB, tD, tR, a);
  return launch_pdl(gemm_kernel<__half>, grid, gm::kThreads, smem, st, "gemm launch", tA, tB, tD, tR, a);
}

int gemm_init() {
  if (int e = check_cuda(cudaFuncSetAttribute(gemm_kernel<__half>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                              gm::kSmemMax),
                         "cudaFuncSetAttribute(gemm)"))
    return e;
  return check_cuda(cudaFuncSetAttribute(gemm_kernel<__nv_bfloat16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         gm::kSmemMax),
                    "cudaFuncSetAttribute(gemm bf16)");
}

}  // namespace wl
