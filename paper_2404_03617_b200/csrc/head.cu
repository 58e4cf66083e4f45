// head.cu — the network's last unit (core.py:144-152; op count
// complexity.py:153-157), which the reference only costs: 1x1 conv to the
// embedding + bias + phi, global average pool, linear classifier.
//   head_pool : one CTA per (image group, embedding chunk of NE columns).
//               The 1x1 conv runs on tcgen05 (M = the group's pixels, N = NE),
//               bias + phi are applied in packed half, the chunk is staged in
//               shared memory and reduced per image by deterministic column
//               sums — the embedding never reaches HBM, only the pooled
//               (n, E) features do.
//   head_fc   : logits = feat W2 + b2, one CTA per (128 batch rows, 32
//               classes), K streamed through a 4-stage TMA / bulk-copy ring.
#include <cuda.h>
#include <cuda_fp16.h>
#include <cstdint>
#include "common.cuh"
#include "plan.h"

namespace wl {

struct HeadArgs {
  int C, E, M, HW, imgs, P, NE, nce;
  int xsw;  // C % 64 == 0: x rows staged as 128-byte swizzled 64-channel blocks (one TMA row per pixel)
  int s_a, s_w, s_st, s_bar, tmem_cols, w1_chunk, o_b1;
  const uint8_t* w1;  // [b1 fp32 E (padded to 128 B)][chunks: NE x C core layout]
  __half* feat;       // (n, E) pooled embedding
};

// Persistent: CTA c owns embedding chunk j = c % nce (its W1 chunk loaded once)
// and loops over image groups g = c / nce, + nsl, ...; x tiles are double
// buffered (TMA), the accumulators double buffered in TMEM, so group g + 1's
// load and 1x1 conv overlap group g's epilogue. Warps 0-7: epilogue (bias +
// phi, staged, per-image column sums); warp 8: loads and MMAs.
constexpr int kHeadThreads = 288;
template <int ACT>
__global__ void __launch_bounds__(kHeadThreads, 1) head_pool_kernel(const __grid_constant__ CUtensorMap tmap_x,
                                                                    const __grid_constant__ HeadArgs a) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* s_w = smem + a.s_w;    // NE x C chunk
  uint8_t* s_st = smem + a.s_st;  // [NE/8][128][8] activated tile
  // bars: 0-1 x_full, 2-3 x_empty, 4-5 acc_full, 6-7 acc_empty, 8 w_full
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + a.s_bar);
  uint32_t* tbase = reinterpret_cast<uint32_t*>(bar + 9);
  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
  const int j = blockIdx.x % a.nce, slice = blockIdx.x / a.nce;
  const int nsl = ((int)gridDim.x - j + a.nce - 1) / a.nce;  // CTAs serving chunk j
  const int groups = (a.P / a.HW + a.imgs - 1) / a.imgs;
  const int my = slice < groups ? (groups - 1 - slice) / nsl + 1 : 0;
  if (tid == 0) {
    for (int i = 0; i < 2; ++i) {
      mbar_init(&bar[i], 1);
      mbar_init(&bar[2 + i], 1);
      mbar_init(&bar[4 + i], 1);
      mbar_init(&bar[6 + i], 256);
    }
    mbar_init(&bar[8], 1);
    fence_mbar_init();
  }
  if (warp == 8) tmem_alloc_n(tbase, a.tmem_cols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  pdl_wait();
  const uint32_t tmem = *tbase;
  if (warp == 8) {
    if (lane == 0) {
      auto load_x = [&](int k) {
        const int b = k & 1, p0 = (slice + k * nsl) * a.imgs * a.HW;
        if (k >= 2) mbar_wait(&bar[2 + b], ((k >> 1) - 1) & 1);
        uint8_t* s_a = smem + a.s_a + b * 128 * a.C * 2;
        mbar_arrive_expect_tx(&bar[b], 128 * a.C * 2);
        if (a.xsw) {
          for (int cb = 0; cb < a.C / 64; ++cb)
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
                "%3}], [%4];" ::"r"(smem_u32(s_a + cb * 16384)),
                "l"(&tmap_x), "r"(cb * 64), "r"(p0), "r"(smem_u32(&bar[b]))
                : "memory");
        } else {
          asm volatile(
              "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, "
              "%4}], [%5];" ::"r"(smem_u32(s_a)),
              "l"(&tmap_x), "r"(0), "r"(p0), "r"(0), "r"(smem_u32(&bar[b]))
              : "memory");
        }
      };
      mbar_arrive_expect_tx(&bar[8], a.w1_chunk);
      bulk_g2s(s_w, a.w1 + align_up(a.E * 4, 128) + (size_t)j * a.w1_chunk, a.w1_chunk, &bar[8]);
      if (my > 0) load_x(0);
      if (my > 1) load_x(1);
      mbar_wait(&bar[8], 0);
      const uint32_t idesc = make_idesc_f16(128, a.NE);
      for (int k = 0; k < my; ++k) {
        const int b = k & 1, u = k >> 1;
        mbar_wait(&bar[b], u & 1);
        mbar_wait(&bar[6 + b], (u & 1) ^ 1);  // the epilogue drained this accumulator
        tc_fence_after();
        const uint32_t sa = smem_u32(smem + a.s_a + b * 128 * a.C * 2);
        for (int kk = 0; kk < a.C / 16; ++kk) {
          const uint64_t ad = a.xsw ? make_sdesc_sw128(sa + (kk / 4) * 16384) + (uint64_t)((kk % 4) * 2)
                                    : make_sdesc(sa + kk * 2 * 2048, 2048, 128);
          const uint64_t bd = make_sdesc(smem_u32(s_w) + kk * 2 * (a.NE * 16), a.NE * 16, 128);
          mma_ss(tmem + b * a.NE, ad, bd, idesc, kk > 0);
        }
        mma_commit(&bar[4 + b]);
        mma_commit(&bar[2 + b]);
        if (k + 2 < my) load_x(k + 2);
      }
    }
  } else {
    const int q = warp % 4, half = warp / 4;
    const float* b1 = reinterpret_cast<const float*>(a.w1) + j * a.NE;
    const int m = q * 32 + lane;
    const float inv = 1.f / (float)a.HW;
    const int i = lane >> 2, w = lane & 3;
    for (int k = 0; k < my; ++k) {
      const int b = k & 1, u = k >> 1, grp = slice + k * nsl;
      mbar_wait(&bar[4 + b], u & 1);
      tc_fence_after();
      for (int c0 = half * 16; c0 < a.NE; c0 += 32) {
        uint32_t v[16];
        WL_TMEM_LD16(tmem_lane_addr(tmem, q, b * a.NE + c0), v);
        tmem_ld_wait();
        *reinterpret_cast<uint4*>(s_st + ((c0 / 8) * 128 + m) * 16) = bias_act8<ACT>(v, b1 + c0);
        *reinterpret_cast<uint4*>(s_st + ((c0 / 8 + 1) * 128 + m) * 16) = bias_act8<ACT>(v + 8, b1 + c0 + 8);
      }
      tc_fence_before();
      mbar_arrive(&bar[6 + b]);
      nbar(1, 256);
      // per-image column sums (fixed order): warp handles 8-channel groups g,
      // lane = (pixel offset i, word w)
      for (int g = warp; g < a.NE / 8; g += 8) {
        const uint8_t* base = s_st + g * 128 * 16 + w * 4;
        for (int im = 0; im < a.imgs; ++im) {
          const int nimg = grp * a.imgs + im;
          float s0 = 0.f, s1 = 0.f;
          for (int p = im * a.HW + i; p < (im + 1) * a.HW; p += 8) {
            const float2 f2 = __half22float2(*reinterpret_cast<const __half2*>(base + p * 16));
            s0 += f2.x;
            s1 += f2.y;
          }
#pragma unroll
          for (int sh = 4; sh < 32; sh <<= 1) {
            s0 += __shfl_xor_sync(0xffffffffu, s0, sh);
            s1 += __shfl_xor_sync(0xffffffffu, s1, sh);
          }
          if (i == 0 && (size_t)nimg * a.HW < (size_t)a.P) {
            __half2 r = __floats2half2_rn(s0 * inv, s1 * inv);
            *reinterpret_cast<__half2*>(a.feat + (size_t)nimg * a.E + j * a.NE + g * 8 + w * 2) = r;
          }
        }
      }
      nbar(1, 256);  // the staging tile is rewritten by the next group
    }
  }
  pdl_trigger();
  tc_fence_before();
  __syncthreads();
  if (warp == 8) tmem_dealloc_n(tmem, a.tmem_cols);
}

struct FcArgs {
  int E, classes, NC, nkc, N, nrows, stages;
  int s_a, s_w, s_bar, tmem_cols, w_chunk;
  const uint8_t* w2;  // [b2 fp32 (padded to 128 B)][class-chunk][k-chunk: NC x 64 core]
  __half* z;          // (n, classes)
};

__global__ void __launch_bounds__(128, 1) head_fc_kernel(const __grid_constant__ CUtensorMap tmap_f,
                                                         const __grid_constant__ FcArgs a) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* s_a = smem + a.s_a;  // stages x [128 rows][64 features], 128B-swizzled (K chunk 64)
  uint8_t* s_w = smem + a.s_w;  // stages x NC x 64
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + a.s_bar);  // full[4], empty[4], mma
  uint32_t* tbase = reinterpret_cast<uint32_t*>(bar + 2 * a.stages + 1);
  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
  const int row0 = (blockIdx.x / a.N) * 128, cc = blockIdx.x % a.N;
  const int S = a.stages;
  if (tid == 0) {
    for (int i = 0; i < 2 * S + 1; ++i) mbar_init(&bar[i], 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc_n(tbase, a.tmem_cols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  pdl_wait();
  const uint32_t tmem = *tbase;
  const uint8_t* wchunks = a.w2 + align_up(a.classes * 4, 128) + (size_t)cc * a.nkc * a.w_chunk;
  if (tid == 0) {
    const uint32_t idesc = make_idesc_f16(128, a.NC);
    auto load = [&](int k) {
      const int b = k % S;
      if (k >= S) mbar_wait(&bar[S + b], ((k / S) - 1) & 1);
      mbar_arrive_expect_tx(&bar[b], 128 * 64 * 2 + a.w_chunk);
      // 64 features x 128 rows as 128-byte swizzled rows (one TMA row per batch row)
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
          "[%4];" ::"r"(smem_u32(s_a + b * 16384)),
          "l"(&tmap_f), "r"(k * 64), "r"(row0), "r"(smem_u32(&bar[b]))
          : "memory");
      bulk_g2s(s_w + b * a.w_chunk, wchunks + (size_t)k * a.w_chunk, a.w_chunk, &bar[b]);
    };
    for (int k = 0; k < S - 1 && k < a.nkc; ++k) load(k);
    for (int k = 0; k < a.nkc; ++k) {
      if (k + S - 1 < a.nkc) load(k + S - 1);
      const int b = k % S;
      mbar_wait(&bar[b], (k / S) & 1);
      tc_fence_after();
      for (int s = 0; s < 4; ++s) {
        const uint64_t ad = make_sdesc_sw128(smem_u32(s_a + b * 16384)) + (uint64_t)(s * 2);
        const uint64_t bd = make_sdesc(smem_u32(s_w + b * a.w_chunk) + s * 2 * (a.NC * 16), a.NC * 16, 128);
        mma_ss(tmem, ad, bd, idesc, (k > 0 || s > 0));
      }
      mma_commit(&bar[S + b]);
    }
    mma_commit(&bar[2 * S]);
  }
  mbar_wait(&bar[2 * S], 0);
  tc_fence_after();
  const float* b2 = reinterpret_cast<const float*>(a.w2);
  const int row = row0 + warp * 32 + lane;
  for (int c0 = 0; c0 < a.NC; c0 += 16) {
    uint32_t v[16];
    WL_TMEM_LD16(tmem_lane_addr(tmem, warp, c0), v);
    tmem_ld_wait();
    if (row >= a.nrows) continue;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const int cls = cc * a.NC + c0 + i;
      if (cls < a.classes) a.z[(size_t)row * a.classes + cls] = __float2half(__uint_as_float(v[i]) + b2[cls]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc_n(tmem, a.tmem_cols);
}

}  // namespace wl

// =================================================================== host
#include <algorithm>
#include <cstring>
#include "gemm.h"
#include "launch.h"

namespace wl {
namespace {

constexpr int kSmemMaxH = 232448;
constexpr int kWsHeader = 4096;  // reserved counter header shared by all families

struct HeadPlan {
  HeadArgs h;
  FcArgs f;
  int64_t w1_bytes, w2_bytes;
  bool fc_gemm;  // classifier on the persistent tcgen05 GEMM (W2^T [classes][E] fp16 + b2)
};

bool head_plan(const wl_block_desc& d, HeadPlan& P) {
  memset(&P, 0, sizeof(P));
  HeadArgs& h = P.h;
  FcArgs& f = P.f;
  h.C = d.c;
  h.E = d.embed;
  h.M = d.classes;
  h.HW = d.h * d.w;
  if (h.C % 16 || h.E % 64 || h.HW > 128 || h.C > 512) return false;
  h.imgs = std::max(1, 128 / h.HW);
  h.xsw = h.C % 64 == 0;
  h.P = d.n * h.HW;
  h.NE = h.E % 128 == 0 ? 128 : 64;  // 96 KB per CTA: two CTAs per SM
  h.nce = h.E / h.NE;
  h.o_b1 = 0;
  h.w1_chunk = h.NE * h.C * 2;
  P.w1_bytes = align_up(h.E * 4, 128) + (int64_t)h.nce * h.w1_chunk;
  int s = 0;
  h.s_a = s;
  s += 2 * 128 * h.C * 2;  // double-buffered x tiles
  h.s_w = s;
  s += h.w1_chunk;
  h.s_st = s;
  s += 128 * h.NE * 2;
  h.s_bar = s;
  if (s + 128 > kSmemMaxH) return false;
  h.tmem_cols = std::max(32, 2 * h.NE);  // double-buffered accumulators
  f.E = h.E;
  f.classes = h.M;
  f.NC = 16;  // 63 class chunks: more CTAs share the K stream
  f.N = (h.M + f.NC - 1) / f.NC;
  f.nkc = h.E / 64;
  f.nrows = d.n;
  f.stages = 8;
  f.w_chunk = f.NC * 64 * 2;
  P.fc_gemm = h.M % 8 == 0 && h.E % 8 == 0;
  P.w2_bytes = P.fc_gemm ? align_up(h.M * 4, 128) + (int64_t)h.M * h.E * 2
                         : align_up(h.M * 4, 128) + (int64_t)f.N * f.nkc * f.w_chunk;
  f.s_a = 0;
  f.s_w = f.stages * 16384;
  f.s_bar = f.s_w + f.stages * f.w_chunk;
  f.tmem_cols = 32;
  return true;
}

using HeadK = void (*)(const CUtensorMap, const HeadArgs);
HeadK head_k(int act) {
  switch (act) {
    case kRelu: return head_pool_kernel<kRelu>;
    case kSilu: return head_pool_kernel<kSilu>;
    case kGelu: return head_pool_kernel<kGelu>;
    case kIdentity: return head_pool_kernel<kIdentity>;
  }
  return nullptr;
}

int head_validate(const wl_block_desc& d) {
  if (d.n < 1 || d.h < 1 || d.w < 1 || d.c < 1) return set_error(WL_EINVAL, "dims must be positive");
  if (d.embed < 1 || d.classes < 1) return set_error(WL_EINVAL, "head widths must be positive");
  if (!head_k(d.act)) return set_error(WL_EUNSUPPORTED, "head activation not supported");
  HeadPlan P;
  if (!head_plan(d, P)) return set_error(WL_EUNSUPPORTED, "no head plan for C=%d %dx%d E=%d", d.c, d.h, d.w, d.embed);
  return WL_OK;
}
int head_wc(const wl_block_desc&) { return 4; }
int64_t head_wn(const wl_block_desc& d, int i) {
  switch (i) {
    case 0: return (int64_t)d.c * d.embed;
    case 1: return d.embed;
    case 2: return (int64_t)d.embed * d.classes;
    case 3: return d.classes;
  }
  return set_error(WL_EINVAL, "weight index out of range");
}
int64_t head_pb(const wl_block_desc& d) {
  HeadPlan P;
  head_plan(d, P);
  return P.w1_bytes + P.w2_bytes;
}
int head_pack(const wl_block_desc& d, const float* const* w, uint8_t* out) {
  HeadPlan P;
  head_plan(d, P);
  const HeadArgs& h = P.h;
  const FcArgs& f = P.f;
  memset(out, 0, (size_t)(P.w1_bytes + P.w2_bytes));
  float* b1 = reinterpret_cast<float*>(out);
  for (int e = 0; e < h.E; ++e) b1[e] = w[1][e];
  uint8_t* c1 = out + align_up(h.E * 4, 128);
  for (int j = 0; j < h.nce; ++j)
    for (int n = 0; n < h.NE; ++n)
      for (int k = 0; k < h.C; ++k)
        put_h(c1 + (size_t)j * h.w1_chunk, core_off_h(n, k, h.NE * 16), w[0][(size_t)k * h.E + j * h.NE + n]);
  uint8_t* o2 = out + P.w1_bytes;
  float* b2 = reinterpret_cast<float*>(o2);
  for (int m = 0; m < h.M; ++m) b2[m] = w[3][m];
  uint8_t* c2 = o2 + align_up(h.M * 4, 128);
  if (P.fc_gemm) {  // W2^T: [classes][E], the GEMM's K-contiguous B operand
    for (int m = 0; m < h.M; ++m)
      for (int e = 0; e < h.E; ++e) put_h(c2, ((size_t)m * h.E + e) * 2, w[2][(size_t)e * h.M + m]);
    return WL_OK;
  }
  for (int cc = 0; cc < f.N; ++cc)
    for (int kc = 0; kc < f.nkc; ++kc) {
      uint8_t* blk = c2 + ((size_t)cc * f.nkc + kc) * f.w_chunk;
      for (int n = 0; n < f.NC; ++n) {
        const int cls = cc * f.NC + n;
        if (cls >= h.M) continue;
        for (int k = 0; k < 64; ++k) put_h(blk, core_off_h(n, k, f.NC * 16), w[2][(size_t)(kc * 64 + k) * h.M + cls]);
      }
    }
  return WL_OK;
}
// workspace: [4 KiB reserved counter header][pooled embedding (n, E) fp16]
int64_t head_ws(const wl_block_desc& d) { return kWsHeader + align_up(d.n * d.embed * 2, 256); }
int head_fwd(const wl_block_desc& d, const void* x, const void* p, void* z, void* ws, cudaStream_t st) {
  HeadPlan P;
  head_plan(d, P);
  HeadArgs h = P.h;
  FcArgs f = P.f;
  uint8_t* feat = reinterpret_cast<uint8_t*>(ws) + kWsHeader;
  CUtensorMap tx, tf;
  {
    if (h.xsw) {
      const uint64_t dims[2] = {(uint64_t)h.C, (uint64_t)h.P};
      const uint64_t strides[1] = {(uint64_t)h.C * 2};
      const uint32_t box[2] = {64, 128};
      if (int e = encode_tmap(&tx, x, 2, dims, strides, box, true)) return e;
    } else {
      const uint64_t dims[3] = {8, (uint64_t)h.P, (uint64_t)(h.C / 8)};
      const uint64_t strides[2] = {(uint64_t)h.C * 2, 16};
      const uint32_t box[3] = {8, 128, (uint32_t)(h.C / 8)};
      if (int e = encode_tmap(&tx, x, 3, dims, strides, box)) return e;
    }
  }
  {
    const uint64_t dims[2] = {(uint64_t)h.E, (uint64_t)d.n};
    const uint64_t strides[1] = {(uint64_t)h.E * 2};
    const uint32_t box[2] = {64, 128};
    if (int e = encode_tmap(&tf, feat, 2, dims, strides, box, true)) return e;
  }
  h.w1 = reinterpret_cast<const uint8_t*>(p);
  h.feat = reinterpret_cast<__half*>(feat);
  const int groups = (d.n + h.imgs - 1) / h.imgs;
  // one CTA per SM at most (persistent over image groups)
  const int grid = std::min(groups * h.nce, std::max(h.nce, kNumSMs));
  if (int e = launch_pdl(head_k(d.act), grid, kHeadThreads, h.s_bar + 128, st, "head_pool launch", tx, h)) return e;
  f.w2 = reinterpret_cast<const uint8_t*>(p) + P.w1_bytes;
  if (P.fc_gemm) {
    GemmEpi ep;
    ep.bias = reinterpret_cast<const float*>(f.w2);
    return gemm_run(feat, d.n, h.E, h.E, f.w2 + align_up(h.M * 4, 128), h.M, h.E, z, h.M, ep, st);
  }
  f.z = reinterpret_cast<__half*>(z);
  const int rows = (d.n + 127) / 128;
  return launch_pdl(head_fc_kernel, rows * f.N, 128, f.s_bar + 256, st, "head_fc launch", tf, f);
}
int head_init() {
  if (int e = gemm_init()) return e;
  for (int act : {kRelu, kSilu, kGelu, kIdentity})
    if (int e = check_cuda(cudaFuncSetAttribute(head_k(act), cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemMaxH),
                           "cudaFuncSetAttribute(head)"))
      return e;
  return check_cuda(cudaFuncSetAttribute(head_fc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemMaxH),
                    "cudaFuncSetAttribute(head_fc)");
}

}  // namespace

const Family kHeadFamily = {head_validate, head_wc, head_wn, head_pb, head_pack, head_ws, head_fwd, head_init};

}  // namespace wl
