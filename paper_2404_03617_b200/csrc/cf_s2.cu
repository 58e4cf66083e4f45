// cf_s2.cu — fused downsampling ConvFirst block on sm_100a.
//
// The reference keeps stride-2 schedules traffic-countable only
// (machine.py:423-425, 476-482) and fixes just the op-count convention
// (complexity.py:185-191): conv at H x W, expansion at H/2 x W, projection at
// H/2 x W/2 -> K. The numerics here follow that convention with BlurPool
// Triangle-3 as the downsampler:
//   xc = conv3x3_T8(x) + b_conv                   (full resolution)
//   xh = blur_H(xc)                               ([1,2,1]/4, stride 2 along H)
//   y  = phi(xh U + a)                            (H/2 x W)
//   yq = blur_W(y)                                (stride 2 along W)
//   z  = yq V + b                                 (H/2 x W/2, K channels)
// One CTA owns R output rows of one image: the x rows it needs arrive by TMA
// in the flat padded layout, the grouped conv runs as block-diagonal
// tcgen05 MMAs, the blurs run on CUDA cores between shared-memory operand
// tiles, expansion (N = hidden chunk) and projection (N = K) run on tcgen05
// with fp32 accumulators in TMEM. Only x and z cross HBM.
#include <cuda.h>
#include <cuda_fp16.h>
#include <cstdint>
#include "common.cuh"
#include "plan.h"

namespace wl {

struct Cf2Args {
  int C, K, hid, r, nch;
  int H, W, Ho, Wo, R, tiles_y, Wp, nbands;
  int n_ct, n_eh, n_pt, conv_base, x_alloc, x_rows, x_bufs;
  int o_convw, o_bconv, o_a, o_b, w_bytes;  // header: conv taps + fp32 vectors
  int chunk_bytes, u_bytes;                 // chunk j = [U_j (r x C) | V_j (K x r)]
  int ws;                                   // 0: every chunk resident; else a ring of ws chunk stages
  int s_x, s_xc, s_ah, s_hs, s_zo, s_aq, s_w, s_bar, smem;
  int ah_bytes, aq_bytes;
  int t_c, t_e, t_z, tmem_cols;
  const uint8_t* wpack;
  __half* z;
  long long* trace;  // debug: clock64 stamps of CTA 0 (null = off)
};

#define CF2_TRACE(slot)                                                          \
  do {                                                                           \
    if (a.trace && blockIdx.x == 0 && (slot) < 256) a.trace[(slot)] = clock64(); \
  } while (0)

// Triangle-3 tap [1, 2, 1] / 4 on 8 packed halves
__device__ __forceinline__ uint4 tri3(const uint4& a, const uint4& b, const uint4& c) {
  uint4 o;
  const __half2* ha = reinterpret_cast<const __half2*>(&a);
  const __half2* hb = reinterpret_cast<const __half2*>(&b);
  const __half2* hc = reinterpret_cast<const __half2*>(&c);
  __half2* ho = reinterpret_cast<__half2*>(&o);
  const __half2 q = __float2half2_rn(0.25f), h = __float2half2_rn(0.5f);
#pragma unroll
  for (int i = 0; i < 4; ++i) ho[i] = __hfma2(hb[i], h, __hmul2(__hadd2(ha[i], hc[i]), q));
  return o;
}

namespace cf2k {
constexpr int kThreads = 640;  // w0 TMA (x bands, weights), w1 FFN MMA, w2/w3 conv MMA (w2 allocates
                               // TMEM), w4-7 conv/blur_H, w8-15 hidden (E -> phi), w16-19 output
                               // (Z -> blur_W)
struct Bars {
  uint64_t w_full, x_full[2], x_empty[2];
  uint64_t conv_full, c_empty, xh_full[2], xh_empty[2];
  uint64_t e_full[2], e_empty[2], q_full[2], q_empty[2];
  uint64_t z_full, z_empty;
  uint64_t wr_full[4], wr_empty[4];
  uint32_t tmem_base;
};
__device__ __forceinline__ void bar_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n)); }
}  // namespace cf2k
__device__ __forceinline__ void tma_store_4d_cf2(const void* tmap, const void* src, int c0, int c1, int c2, int c3) {
  asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%2, %3, %4, %5}], [%1];" ::"l"(tmap),
               "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
               : "memory");
}
__device__ __forceinline__ void bulk_commit_cf2() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0_cf2() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all_cf2() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
namespace cf2k {
}  // namespace cf2k

// Persistent CTA over bands of R output rows; the stages of consecutive bands
// overlap: the tensor core runs the conv of band i+1 and the expand/project
// chunks of band i while the CUDA-core warp groups drain the accumulators.
// BlurPool along W commutes with the (linear) projection, so it is applied to
// the K-channel projection output instead of the hidden activation:
//   z = blur_W(y) V + b = blur_W(y V) + b     (y = phi(xh U + a))
// which keeps the hidden-side CUDA-core work to one drain per chunk.
template <int ACT>
__global__ void __launch_bounds__(cf2k::kThreads, 1)
    cf2_kernel(const __grid_constant__ CUtensorMap tmap_x, const __grid_constant__ CUtensorMap tmap_z,
               const __grid_constant__ Cf2Args a) {
  using namespace cf2k;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* s_x = smem + a.s_x;
  __half* s_xc = reinterpret_cast<__half*>(smem + a.s_xc);
  uint8_t* s_ah = smem + a.s_ah;
  __half* s_zs = reinterpret_cast<__half*>(smem + a.s_hs);
  __half* s_zo = reinterpret_cast<__half*>(smem + a.s_zo);
  uint8_t* s_aq = smem + a.s_aq;
  uint8_t* s_w = smem + a.s_w;
  Bars& B = *reinterpret_cast<Bars*>(smem + a.s_bar);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int C = a.C, K = a.K, r = a.r, W = a.W, Wp = a.Wp, nch = a.nch;
  const int planes = C / 8;
  const int loaded = a.x_rows * Wp;
  const int MH = a.n_eh * 128;
  const int RW = a.R * W;
  const int nb = a.nbands > (int)blockIdx.x ? (a.nbands - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
  auto band_of = [&](int i) { return (int)blockIdx.x + i * (int)gridDim.x; };

  // zero the conv-tile overrun past the loaded rows (TMA never writes it)
  for (int xb = 0; xb < a.x_bufs; ++xb)
    for (int i = threadIdx.x; i < planes * (a.x_alloc - loaded); i += blockDim.x) {
      const int pl = i / (a.x_alloc - loaded), f = loaded + i % (a.x_alloc - loaded);
      *reinterpret_cast<uint4*>(s_x + ((size_t)(xb * planes + pl) * a.x_alloc + f) * 16) = make_uint4(0, 0, 0, 0);
    }
  if (threadIdx.x == 0) {
    mbar_init(&B.w_full, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&B.x_full[i], 1);
      mbar_init(&B.x_empty[i], 2);
      mbar_init(&B.xh_full[i], 128);
      mbar_init(&B.xh_empty[i], 1);
      mbar_init(&B.e_full[i], 1);
      mbar_init(&B.e_empty[i], 256);
      mbar_init(&B.q_full[i], 256);
      mbar_init(&B.q_empty[i], 1);
    }
    mbar_init(&B.conv_full, 2);
    mbar_init(&B.c_empty, 128);
    mbar_init(&B.z_full, 1);
    mbar_init(&B.z_empty, 128);
    for (int i = 0; i < 4; ++i) {
      mbar_init(&B.wr_full[i], 1);
      mbar_init(&B.wr_empty[i], 1);
    }
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc_n(&B.tmem_base, a.tmem_cols);
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  pdl_trigger();  // single-wave persistent grid: let the next kernel stage its prologue
  pdl_wait();
  const uint32_t tmem = B.tmem_base;
  if (threadIdx.x == 0) CF2_TRACE(0);

  if (warp == 0) {
    // ---------------- producer: resident weights once, x bands through a ring
    if (lane == 0) {
      prefetch_tmap(&tmap_x);
      const int wtot = a.w_bytes + (a.ws ? 0 : nch * a.chunk_bytes);
      mbar_arrive_expect_tx(&B.w_full, wtot);
      bulk_g2s(s_w, a.wpack, wtot, &B.w_full);
      auto load_x = [&](int i) {
        const int xb = i % a.x_bufs;
        if (i < 8) CF2_TRACE(8 + i * 24 + 0);
        const int band = band_of(i), n = band / a.tiles_y, yo0 = (band % a.tiles_y) * a.R;
        mbar_arrive_expect_tx(&B.x_full[xb], planes * loaded * 16);
        for (int g = 0; g < planes; ++g)
          tma_load_5d(s_x + ((size_t)(xb * planes + g) * a.x_alloc) * 16, &tmap_x, 0, -1, 2 * yo0 - 2, g, n,
                      &B.x_full[xb]);
      };
      if (!a.ws) {
        for (int i = 0; i < nb; ++i) {
          mbar_wait_sleep(&B.x_empty[i % a.x_bufs], ((i / a.x_bufs) & 1) ^ 1);
          load_x(i);
        }
      } else {
        // streamed FFN weights: x bands and weight chunks from one thread,
        // each issued as soon as its ring slot frees (neither waits behind the other)
        const uint8_t* chunks = a.wpack + a.w_bytes;
        const int total = nb * nch;
        int i = 0, g = 0;
        while (i < nb || g < total) {
          bool moved = false;
          if (i < nb && mbar_test(&B.x_empty[i % a.x_bufs], ((i / a.x_bufs) & 1) ^ 1)) {
            load_x(i++);
            moved = true;
          }
          if (g < total && mbar_test(&B.wr_empty[g % a.ws], ((g / a.ws) & 1) ^ 1)) {
            const int slot = g % a.ws;
            mbar_arrive_expect_tx(&B.wr_full[slot], a.chunk_bytes);
            bulk_g2s(s_w + a.w_bytes + slot * a.chunk_bytes, chunks + (size_t)(g % nch) * a.chunk_bytes,
                     a.chunk_bytes, &B.wr_full[slot]);
            ++g;
            moved = true;
          }
          if (!moved) __nanosleep(32);
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer
    {  // warp-converged issue: one elected lane issues each MMA / commit
      mbar_wait(&B.w_full, 0);
      const uint32_t cw = smem_u32(s_w + a.o_convw);
      const uint32_t idesc_c = make_idesc_f16(128, 16);
      const uint32_t idesc_e = make_idesc_f16(128, r);
      const uint32_t idesc_z = make_idesc_f16(128, K);
      auto conv_begin = [&](int i) {
        if (i < 8) if (lane == 0) CF2_TRACE(8 + i * 24 + 1);
        mbar_wait(&B.x_full[i % a.x_bufs], (i / a.x_bufs) & 1);
        mbar_wait(&B.c_empty, (i & 1) ^ 1);  // previous band's conv accumulators drained
        tc_fence_after();
        if (i < 8) if (lane == 0) CF2_TRACE(8 + i * 24 + 2);
      };
      auto conv_tiles = [&](int i, int t0, int t1) {
        const uint32_t x0 = smem_u32(s_x) + (i % a.x_bufs) * planes * a.x_alloc * 16;
        for (int t = t0; t < t1; ++t)
          for (int pr = 0; pr < C / 16; ++pr) {
            const uint64_t ad = make_sdesc(x0 + (2 * pr * a.x_alloc + a.conv_base - Wp - 1 + t * 128) * 16,
                                           a.x_alloc * 16, 128);
            uint64_t aa = ad, bd = make_sdesc(cw + pr * 9 * 512, 256, 128);
            const uint32_t d = tmem + a.t_c + t * C + 16 * pr;
#pragma unroll
            for (int tap = 0; tap < 9; ++tap) {  // incremental descriptors (cheap issue)
              mma_ss_w(d, aa, bd, idesc_c, tap > 0);
              aa += (tap % 3 == 2) ? (uint64_t)(Wp - 2) : 1ull;
              bd += 32;
            }
          }
      };
      auto conv_end = [&](int i) {
        mma_commit_w(&B.conv_full);
        mma_commit_w(&B.x_empty[i % a.x_bufs]);
        if (i < 8) if (lane == 0) CF2_TRACE(8 + i * 24 + 3);
      };
      // chunk j of band i (global index g): resident slot j, or ring stage g % ws
      auto chunk_addr = [&](int g, int j) -> uint32_t {
        return smem_u32(s_w) + a.w_bytes + (a.ws ? g % a.ws : j) * a.chunk_bytes;
      };
      auto issue_project = [&](int i, int j) {
        const int gq = i * nch + j, qs = gq & 1;
        mbar_wait(&B.q_full[qs], (gq >> 1) & 1);
        if (j == 0) mbar_wait(&B.z_empty, (i & 1) ^ 1);
        tc_fence_after();
        const uint32_t vb = chunk_addr(gq, j) + a.u_bytes;
        const uint32_t aq = smem_u32(s_aq) + qs * a.aq_bytes;
        for (int t = 0; t < a.n_eh; ++t)
          for (int kk = 0; kk < r / 16; ++kk)
            mma_ss_w(tmem + a.t_z + t * K, make_sdesc(aq + (kk * 2 * MH + t * 128) * 16, MH * 16, 128),
                   make_sdesc(vb + kk * 2 * (K * 16), K * 16, 128), idesc_z, (j > 0 || kk > 0));
        mma_commit_w(&B.q_empty[qs]);
        if (a.ws) mma_commit_w(&B.wr_empty[gq % a.ws]);
        if (j == nch - 1) mma_commit_w(&B.z_full);
      };
      // warp 1 issues the FFN (expand / project chunks); the grouped conv is
      // issued by warps 3 and 2 (below) and runs ahead as far as G1's drain
      // of the single conv accumulator allows
      for (int i = 0; i < nb; ++i) {
        const int hb = i & 1;
        mbar_wait(&B.xh_full[hb], (i >> 1) & 1);
        tc_fence_after();
        if (i < 8) if (lane == 0) CF2_TRACE(8 + i * 24 + 4);
        const uint32_t ah = smem_u32(s_ah) + hb * a.ah_bytes;
        for (int j = 0; j < nch; ++j) {
          const int gg = i * nch + j, es = gg & 1;
          mbar_wait(&B.e_empty[es], ((gg >> 1) & 1) ^ 1);
          if (a.ws) mbar_wait(&B.wr_full[gg % a.ws], (gg / a.ws) & 1);
          tc_fence_after();
          const uint32_t ub = chunk_addr(gg, j);
          for (int t = 0; t < a.n_eh; ++t)
            for (int kk = 0; kk < C / 16; ++kk)
              mma_ss_w(tmem + a.t_e + (es * a.n_eh + t) * r, make_sdesc(ah + (kk * 2 * MH + t * 128) * 16, MH * 16, 128),
                     make_sdesc(ub + kk * 2 * (r * 16), r * 16, 128), idesc_e, kk > 0);
          mma_commit_w(&B.e_full[es]);
          if (j == nch - 1) mma_commit_w(&B.xh_empty[hb]);
          if (j > 0) issue_project(i, j - 1);
        }
        issue_project(i, nch - 1);
        if (i < 8) if (lane == 0) CF2_TRACE(8 + i * 24 + 5);
      }
    }
  } else if (warp == 3 || warp == 2) {
    // ---------------- grouped-conv issuers: conv tiles split between two threads
    {  // warp-converged issue: one elected lane issues each MMA / commit
      const int ci = warp == 3 ? 0 : 1;
      mbar_wait(&B.w_full, 0);
      const uint32_t cw = smem_u32(s_w + a.o_convw);
      const uint32_t idesc_c = make_idesc_f16(128, 16);
      for (int i = 0; i < nb; ++i) {
        const int xb = i % a.x_bufs;
        mbar_wait(&B.x_full[xb], (i / a.x_bufs) & 1);
        mbar_wait(&B.c_empty, (i & 1) ^ 1);  // previous band's conv accumulators drained
        tc_fence_after();
        if (ci == 0 && i < 8) if (lane == 0) CF2_TRACE(8 + i * 24 + 2);
        const uint32_t x0 = smem_u32(s_x) + xb * planes * a.x_alloc * 16;
        for (int t = ci; t < a.n_ct; t += 2)
          for (int pr = 0; pr < C / 16; ++pr) {
            uint64_t aa = make_sdesc(x0 + (2 * pr * a.x_alloc + a.conv_base - Wp - 1 + t * 128) * 16, a.x_alloc * 16, 128);
            uint64_t bd = make_sdesc(cw + pr * 9 * 512, 256, 128);
            const uint32_t d = tmem + a.t_c + t * C + 16 * pr;
#pragma unroll
            for (int tap = 0; tap < 9; ++tap) {
              mma_ss_w(d, aa, bd, idesc_c, tap > 0);
              aa += (tap % 3 == 2) ? (uint64_t)(Wp - 2) : 1ull;
              bd += 32;
            }
          }
        mma_commit_w(&B.conv_full);
        mma_commit_w(&B.x_empty[xb]);
        if (ci == 0 && i < 8) if (lane == 0) CF2_TRACE(8 + i * 24 + 3);
      }
    }
  } else if (warp >= 4 && warp < 8) {
    // ---------------- conv drain (+ b_conv -> fp16 xc planes) and blur along H -> expand operand
    const int q = warp % 4, tid = threadIdx.x - 128;
    mbar_wait_sleep(&B.w_full, 0);
    const float* bconv = reinterpret_cast<const float*>(s_w + a.o_bconv);
    const int XP = (2 * a.R + 1) * W;
    const int cb = C / 16;  // 16-column blocks per conv tile
    float bc[2][16];
#pragma unroll
    for (int b = 0; b < 2; ++b)
#pragma unroll
      for (int k = 0; k < 16; ++k) bc[b][k] = b < cb ? bconv[b * 16 + k] : 0.f;
    for (int i = 0; i < nb; ++i) {
      const int band = band_of(i), yo0 = (band % a.tiles_y) * a.R;
      mbar_wait_sleep(&B.conv_full, i & 1);
      tc_fence_after();
      if (tid == 0 && i < 8) CF2_TRACE(8 + i * 24 + 6);
      // lane row -> (flat row, col) walked incrementally (no integer division per tile)
      int row = (a.conv_base + q * 32 + lane) / Wp, col = a.conv_base + q * 32 + lane - row * Wp;
      for (int t = 0; t < a.n_ct; ++t) {
        const bool inside = col >= 1 && col <= W && row >= 1 && row <= 2 * a.R + 1;  // row 1 .. 2R+1 <-> conv row 2*yo0 - 2 + row
        const int px = (row - 1) * W + (col - 1);
        for (int b0 = 0; b0 < cb; b0 += 2) {  // 32 columns per TMEM round trip
          uint32_t v[2][16];
          WL_TMEM_LD16(tmem_lane_addr(tmem, q, a.t_c + t * C + 16 * b0), v[0]);
          if (b0 + 1 < cb) WL_TMEM_LD16(tmem_lane_addr(tmem, q, a.t_c + t * C + 16 * b0 + 16), v[1]);
          tmem_ld_wait();
          if (inside) {
#pragma unroll
            for (int b = 0; b < 2; ++b) {
              if (b0 + b >= cb) break;
              float fv[16];
              if (b0 == 0) {
#pragma unroll
                for (int k = 0; k < 16; ++k) fv[k] = __uint_as_float(v[b][k]) + bc[b][k];
              } else {  // C > 32: the other channel blocks' biases come from shared memory
#pragma unroll
                for (int k = 0; k < 16; ++k) fv[k] = __uint_as_float(v[b][k]) + bconv[(b0 + b) * 16 + k];
              }
              const int pl = 2 * (b0 + b);
              *reinterpret_cast<uint4*>(s_xc + ((size_t)pl * XP + px) * 8) = pack8(fv);
              *reinterpret_cast<uint4*>(s_xc + ((size_t)(pl + 1) * XP + px) * 8) = pack8(fv + 8);
            }
          }
        }
        col += 128;
        while (col >= Wp) {
          col -= Wp;
          ++row;
        }
      }
      tc_fence_before();
      mbar_arrive(&B.c_empty);
      if (tid == 0 && i < 8) CF2_TRACE(8 + i * 24 + 7);
      const int hb = i & 1;
      mbar_wait_sleep(&B.xh_empty[hb], ((i >> 1) & 1) ^ 1);
      bar_sync(1, 128);  // all of xc written
      uint8_t* ah = s_ah + hb * a.ah_bytes;
      for (int c8 = 0; c8 < planes; ++c8) {
        const __half* plc = s_xc + (size_t)c8 * XP * 8;
        uint8_t* ahc = ah + (size_t)c8 * MH * 16;
        int ro = tid / W, x = tid - ro * W;
        for (int p = tid; p < RW; p += 128) {
          const int k0 = (yo0 + ro == 0) ? 2 : 2 * ro;  // xc rows of conv rows 2yo-1 (reflect -1 -> 1), 2yo, 2yo+1
          const __half* pl = plc + (size_t)x * 8;
          *reinterpret_cast<uint4*>(ahc + (size_t)p * 16) =
              tri3(lds128(pl + (size_t)k0 * W * 8), lds128(pl + (size_t)(2 * ro + 1) * W * 8),
                   lds128(pl + (size_t)(2 * ro + 2) * W * 8));  // explicit 16-byte loads (no 4x split)
          x += 128;
          while (x >= W) {
            x -= W;
            ++ro;
          }
        }
      }
      fence_async_smem();
      mbar_arrive(&B.xh_full[hb]);
      if (tid == 0 && i < 8) CF2_TRACE(8 + i * 24 + 8);
      bar_sync(1, 128);  // xc free for the next band
    }
  } else if (warp >= 8 && warp < 16) {
    // ---------------- hidden chunks: E + a -> phi -> fp16 project operand planes
    // (two warps per TMEM quadrant, alternating 32-column blocks)
    const int q = warp % 4, hh = (warp - 8) / 4, tid = threadIdx.x - 256;
    mbar_wait_sleep(&B.w_full, 0);
    const float* av = reinterpret_cast<const float*>(s_w + a.o_a);
    for (int i = 0; i < nb; ++i) {
      for (int j = 0; j < nch; ++j) {
        const int gg = i * nch + j, es = gg & 1;
        mbar_wait_sleep(&B.e_full[es], (gg >> 1) & 1);
        mbar_wait_sleep(&B.q_empty[es], ((gg >> 1) & 1) ^ 1);
        tc_fence_after();
        if (tid == 0 && i < 8 && j < 4) CF2_TRACE(8 + i * 24 + 9 + 3 * j);
        uint8_t* aq = s_aq + es * a.aq_bytes;
        const float* avj = av + j * r;
        for (int t = 0; t < a.n_eh; ++t) {
          const int p = t * 128 + q * 32 + lane;
          const uint32_t tcol = a.t_e + (es * a.n_eh + t) * r;
          // 16-column blocks alternate between the two warps of a quadrant (both
          // busy for any chunk width r >= 32); biases are two vector loads each
          for (int c0 = hh * 16; c0 < r; c0 += 32) {
            uint32_t v[16];
            WL_TMEM_LD16(tmem_lane_addr(tmem, q, tcol + c0), v);
            tmem_ld_wait();
            *reinterpret_cast<uint4*>(aq + ((size_t)(c0 / 8) * MH + p) * 16) = bias_act8<ACT>(v, avj + c0);
            *reinterpret_cast<uint4*>(aq + ((size_t)(c0 / 8 + 1) * MH + p) * 16) = bias_act8<ACT>(v + 8, avj + c0 + 8);
          }
        }
        tc_fence_before();
        mbar_arrive(&B.e_empty[es]);
        fence_async_smem();
        mbar_arrive(&B.q_full[es]);
        if (tid == 0 && i < 8 && j < 4) CF2_TRACE(8 + i * 24 + 11 + 3 * j);
      }
    }
  } else if (warp >= 16) {
    // ---------------- output: Z + b -> fp16 staging -> blur along W (stride 2) -> TMA store
    const int q = warp % 4, tid = threadIdx.x - 512;
    mbar_wait_sleep(&B.w_full, 0);
    const float* bv = reinterpret_cast<const float*>(s_w + a.o_b);
    const int k8 = K / 8, KP = K + 8;
    const int RWo = a.R * a.Wo;
    for (int i = 0; i < nb; ++i) {
      const int band = band_of(i), n = band / a.tiles_y, yo0 = (band % a.tiles_y) * a.R;
      mbar_wait_sleep(&B.z_full, i & 1);
      tc_fence_after();
      if (tid == 0 && i < 8) CF2_TRACE(8 + i * 24 + 21);
      // staging: pixel-major rows of KP = K + 8 halves (the 16-byte pad spreads
      // a warp's row-strided stores over the banks)
      for (int t = 0; t < a.n_eh; ++t) {
        const int p = t * 128 + q * 32 + lane;
        for (int c0 = 0; c0 < K; c0 += 32) {
          uint32_t v[2][16];
          const bool two = c0 + 16 < K;
          WL_TMEM_LD16(tmem_lane_addr(tmem, q, a.t_z + t * K + c0), v[0]);
          if (two) WL_TMEM_LD16(tmem_lane_addr(tmem, q, a.t_z + t * K + c0 + 16), v[1]);
          tmem_ld_wait();
          if (p >= RW) continue;
#pragma unroll
          for (int b = 0; b < 2; ++b) {
            if (b == 1 && !two) break;
            const int cc = c0 + 16 * b;
            float fv[16], b16[16];
            load16f(bv + cc, b16);
#pragma unroll
            for (int k = 0; k < 16; ++k) fv[k] = __uint_as_float(v[b][k]) + b16[k];
            *reinterpret_cast<uint4*>(s_zs + (size_t)p * KP + cc) = pack8(fv);
            *reinterpret_cast<uint4*>(s_zs + (size_t)p * KP + cc + 8) = pack8(fv + 8);
          }
        }
      }
      tc_fence_before();
      mbar_arrive(&B.z_empty);
      if (tid == 0) bulk_wait_read0_cf2();  // previous band's store has left the output staging
      bar_sync(3, 128);                     // staging complete
      // output pixel qi = (ro, xo), 8-channel group c8; items ordered c8-fastest
      // so a warp writes contiguous 16-byte chunks of the dense [R][Wo][K] tile
      {
        int c8 = tid % k8, qi = tid / k8;
        const int sq = 128 / k8, sc = 128 % k8;
        int ro = qi / a.Wo, xo = qi - ro * a.Wo;
        for (int idx = tid; idx < RWo * k8; idx += 128) {
          const int x0 = xo == 0 ? 1 : 2 * xo - 1;  // reflect column -1 -> 1
          const __half* rb = s_zs + (size_t)ro * W * KP + c8 * 8;
          *reinterpret_cast<uint4*>(s_zo + ((size_t)qi * K + c8 * 8)) =
              tri3(lds128(rb + (size_t)x0 * KP), lds128(rb + (size_t)(2 * xo) * KP),
                   lds128(rb + (size_t)(2 * xo + 1) * KP));
          c8 += sc;
          int dq = sq;
          if (c8 >= k8) {
            c8 -= k8;
            ++dq;
          }
          qi += dq;
          xo += dq;
          while (xo >= a.Wo) {
            xo -= a.Wo;
            ++ro;
          }
        }
      }
      fence_async_smem();
      bar_sync(3, 128);
      if (tid == 0) {
        tma_store_4d_cf2(&tmap_z, s_zo, 0, 0, yo0, n);
        bulk_commit_cf2();
      }
      if (tid == 0 && i < 8) CF2_TRACE(8 + i * 24 + 22);
      bar_sync(3, 128);  // staging free for the next band
    }
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) {
    CF2_TRACE(1);
    if (a.trace && blockIdx.x == 0) {
      a.trace[2] = a.R * 1000 + a.r;
      a.trace[3] = a.n_ct * 10000 + a.n_eh * 100 + a.n_pt;
      a.trace[4] = nb * 10 + a.x_bufs;
    }
  }
  if (warp == 16 && lane == 0) bulk_wait_all_cf2();  // output stores complete before exit
  if (warp == 2) tmem_dealloc_n(tmem, a.tmem_cols);
}

}  // namespace wl

// =================================================================== host
#include <algorithm>
#include <cstring>
#include <cstdlib>
#include "launch.h"

namespace wl {
namespace {

constexpr int kSmemMax2 = 232448;
long long* g_cf2_trace = nullptr;

bool cf2_plan(const wl_block_desc& d, Cf2Args& a) {
  memset(&a, 0, sizeof(a));
  a.C = d.c;
  a.K = d.k;
  a.hid = d.expansion * d.c;
  a.H = d.h;
  a.W = d.w;
  a.Ho = d.h / 2;
  a.Wo = d.w / 2;
  a.Wp = d.w + 1;
  if (a.C % 16 || a.K % 16 || a.hid % 16 || a.K > 256) return false;
  // choose (R output rows per band, hidden chunk r, x buffers) by the
  // tcgen05 cost model (max(44, N/2) cycles per K=16 instruction) per output
  // row, subject to TMEM (512 columns) and shared memory
  double best = 1e30;
  Cf2Args bestA{};
  // planner experiments: WL_CF2_R pins the band height (read once per process)
  static const char* force_r = [] {
    const char* e = getenv("WL_CF2_R");
    return e && *e ? e : nullptr;  // empty = unset
  }();
  for (int R = 1; R <= 8; ++R) {
    if (R > a.Ho) break;
    // measured: bands wider than 256 pixels lengthen each band's chain, and odd
    // heights above 1 run 1.4-2x slower than their even neighbours (W = 56 and 112)
    if (force_r ? R != atoi(force_r) : R > 1 && (R * a.W > 256 || R % 2)) continue;
    for (int rr = 16; rr <= 256 && rr <= a.hid; rr += 16) {
      if (a.hid % rr) continue;
      for (int xbufs = 2; xbufs >= 1; --xbufs)
      for (int ws : {0, 3, 2}) {
        Cf2Args c = a;
        c.ws = ws;
        c.R = R;
        c.r = rr;
        c.nch = c.hid / rr;
        c.x_bufs = xbufs;
        c.x_rows = 2 * R + 3;
        c.conv_base = c.Wp + 1;
        const int conv_end = (2 * R + 2) * c.Wp;
        c.n_ct = (conv_end - c.conv_base + 127) / 128;
        c.x_alloc = align_up(std::max(c.conv_base + c.n_ct * 128 + c.Wp + 2, c.x_rows * c.Wp), 8);
        c.n_eh = (R * c.W + 127) / 128;
        c.n_pt = c.n_eh;  // the projection runs at (R, W); BlurPool W follows it
        c.t_c = 0;
        c.t_e = c.n_ct * c.C;
        c.t_z = c.t_e + 2 * c.n_eh * rr;
        const int cols = c.t_z + c.n_pt * c.K;
        if (cols > 512) continue;
        int o = 0;
        c.o_convw = o;
        o += (c.C / 16) * 9 * 512;
        c.o_bconv = o;
        o = align_up(o + c.C * 4, 16);
        c.o_a = o;
        o = align_up(o + c.hid * 4, 16);
        c.o_b = o;
        o = align_up(o + c.K * 4, 16);
        c.w_bytes = align_up(o, 128);
        c.u_bytes = rr * c.C * 2;
        c.chunk_bytes = c.u_bytes + c.K * rr * 2;
        c.ah_bytes = c.n_eh * 128 * c.C * 2;
        c.aq_bytes = c.n_eh * 128 * rr * 2;
        int s = 0;
        c.s_x = s;
        s = align_up(s + xbufs * (c.C / 8) * c.x_alloc * 16, 128);
        c.s_xc = s;
        s = align_up(s + (2 * R + 1) * c.W * c.C * 2, 128);
        c.s_ah = s;
        s = align_up(s + 2 * c.ah_bytes, 128);
        c.s_hs = s;  // projection staging (pixel-major rows of K + 8 halves) for BlurPool W
        s = align_up(s + R * c.W * (c.K + 8) * 2, 128);
        c.s_zo = s;  // dense output tile [R][Wo][K] for the TMA store
        s = align_up(s + R * c.Wo * c.K * 2, 128);
        c.s_aq = s;
        s = align_up(s + 2 * c.aq_bytes, 128);
        c.s_w = s;
        s = align_up(s + c.w_bytes + (ws ? std::min(ws, c.nch) : c.nch) * c.chunk_bytes, 128);
        if (ws > c.nch) continue;
        c.s_bar = s;
        s += 256;
        c.smem = s;
        if (s > kSmemMax2) continue;
        const double conv = (double)c.n_ct * (c.C / 16) * 9 * 44;
        const double expand = (double)c.n_eh * (c.C / 16) * c.nch * std::max(44, rr / 2);
        const double project = (double)c.n_pt * (c.hid / 16) * std::max(44, c.K / 2);
        // TMEM reads of the accumulators (~128 B/cycle): conv, hidden, projection
        const double tmem_rd = 4.0 * ((double)c.n_ct * c.C + (double)c.n_eh * c.hid + (double)c.n_pt * c.K);
        // streamed plans re-read every chunk per band from L2 (~50 B/cycle)
        const double l2 = ws ? (double)c.nch * c.chunk_bytes / 50.0 : 0.0;
        const double cost = (std::max(std::max(conv + expand + project, tmem_rd), l2) + 300.0 + (ws ? 200.0 : 0.0)) / R *
                            (xbufs == 2 ? 1.0 : 1.15);
        if (cost < best) {
          best = cost;
          bestA = c;
        }
      }
    }
  }
  if (best >= 1e30) return false;
  a = bestA;
  a.tiles_y = (a.Ho + a.R - 1) / a.R;
  a.nbands = d.n * a.tiles_y;
  a.tmem_cols = 32;
  while (a.tmem_cols < a.t_z + a.n_pt * a.K) a.tmem_cols *= 2;
  return true;
}

using Cf2K = void (*)(const CUtensorMap, const CUtensorMap, const Cf2Args);
Cf2K cf2_kernel_for(int act) {
  switch (act) {
    case kRelu: return cf2_kernel<kRelu>;
    case kSilu: return cf2_kernel<kSilu>;
    case kGelu: return cf2_kernel<kGelu>;
  }
  return nullptr;
}

int cf2_validate(const wl_block_desc& d) {
  if (d.h % 2 || d.w % 2) return set_error(WL_EINVAL, "stride 2 needs an even resolution");
  if (d.group_width != 8 || d.ksize != 3)
    return set_error(WL_EUNSUPPORTED, "downsampling ConvFirst supports T=8 3x3 (got T=%d k=%d)", d.group_width, d.ksize);
  if (d.norm != WL_NORM_NONE) return set_error(WL_EUNSUPPORTED, "downsampling ConvFirst has no norm");
  if (!cf2_kernel_for(d.act)) return set_error(WL_EUNSUPPORTED, "activation not supported");
  Cf2Args a;
  if (!cf2_plan(d, a)) return set_error(WL_EUNSUPPORTED, "no launch plan for downsampling ConvFirst C=%d K=%d", d.c, d.k);
  return WL_OK;
}
int cf2_weight_count(const wl_block_desc&) { return 6; }
int64_t cf2_weight_numel(const wl_block_desc& d, int i) {
  const int64_t c = d.c, hid = (int64_t)d.expansion * d.c, k = d.k;
  switch (i) {
    case 0: return c * 9 * d.group_width;
    case 1: return c;
    case 2: return c * hid;
    case 3: return hid;
    case 4: return hid * k;
    case 5: return k;
  }
  return set_error(WL_EINVAL, "weight index %d out of range", i);
}
int64_t cf2_packed_bytes(const wl_block_desc& d) {
  Cf2Args a;
  cf2_plan(d, a);
  return a.w_bytes + (int64_t)a.nch * a.chunk_bytes;
}
int cf2_pack(const wl_block_desc& d, const float* const* w, uint8_t* out) {
  Cf2Args a;
  cf2_plan(d, a);
  memset(out, 0, (size_t)cf2_packed_bytes(d));
  const int C = a.C, hid = a.hid, K = a.K, r = a.r;
  const float *wc = w[0], *bc = w[1], *u = w[2], *av = w[3], *v = w[4], *b = w[5];
  for (int pr = 0; pr < C / 16; ++pr)
    for (int t = 0; t < 9; ++t)
      for (int nn = 0; nn < 16; ++nn)
        for (int kk = 0; kk < 16; ++kk) {
          if (nn / 8 != kk / 8) continue;
          put_h(out + a.o_convw + (pr * 9 + t) * 512, core_off_h(nn, kk, 256), wc[((size_t)(16 * pr + nn) * 9 + t) * 8 + kk % 8]);
        }
  float* fb = reinterpret_cast<float*>(out + a.o_bconv);
  float* fa = reinterpret_cast<float*>(out + a.o_a);
  float* fbb = reinterpret_cast<float*>(out + a.o_b);
  for (int i = 0; i < C; ++i) fb[i] = bc[i];
  for (int i = 0; i < hid; ++i) fa[i] = av[i];
  for (int i = 0; i < K; ++i) fbb[i] = b[i];
  for (int j = 0; j < a.nch; ++j) {
    uint8_t* ub = out + a.w_bytes + (size_t)j * a.chunk_bytes;
    for (int nn = 0; nn < r; ++nn)
      for (int k = 0; k < C; ++k) put_h(ub, core_off_h(nn, k, r * 16), u[(size_t)k * hid + j * r + nn]);
    uint8_t* vb = ub + a.u_bytes;
    for (int nn = 0; nn < K; ++nn)
      for (int k = 0; k < r; ++k) put_h(vb, core_off_h(nn, k, K * 16), v[(size_t)(j * r + k) * K + nn]);
  }
  return WL_OK;
}
int64_t cf2_ws(const wl_block_desc&) { return 0; }
int cf2_forward(const wl_block_desc& d, const void* x, const void* packed, void* z, void*, cudaStream_t st) {
  Cf2Args a;
  cf2_plan(d, a);
  CUtensorMap tm;
  const uint64_t dims[5] = {8, (uint64_t)d.w, (uint64_t)d.h, (uint64_t)(d.c / 8), (uint64_t)d.n};
  const uint64_t strides[4] = {(uint64_t)d.c * 2, (uint64_t)d.w * d.c * 2, 16, (uint64_t)d.h * d.w * d.c * 2};
  const uint32_t box[5] = {8, (uint32_t)a.Wp, (uint32_t)a.x_rows, 1, 1};
  if (int e = encode_tmap(&tm, x, 5, dims, strides, box)) return e;
  CUtensorMap tz;
  const uint64_t zd[4] = {(uint64_t)d.k, (uint64_t)a.Wo, (uint64_t)a.Ho, (uint64_t)d.n};
  const uint64_t zs[3] = {(uint64_t)d.k * 2, (uint64_t)a.Wo * d.k * 2, (uint64_t)a.Ho * a.Wo * d.k * 2};
  const uint32_t zb[4] = {(uint32_t)d.k, (uint32_t)a.Wo, (uint32_t)a.R, 1};
  if (int e = encode_tmap(&tz, z, 4, zd, zs, zb)) return e;
  a.wpack = reinterpret_cast<const uint8_t*>(packed);
  a.z = reinterpret_cast<__half*>(z);
  a.trace = g_cf2_trace;
  const int grid = std::min(a.nbands, kNumSMs);
  return launch_pdl(cf2_kernel_for(d.act), grid, cf2k::kThreads, a.smem, st, "cf2 launch", tm, tz, a);
}
int cf2_init() {
  for (int act : {kRelu, kSilu, kGelu})
    if (int e = check_cuda(cudaFuncSetAttribute(cf2_kernel_for(act), cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemMax2),
                           "cudaFuncSetAttribute(cf2)"))
      return e;
  return WL_OK;
}

}  // namespace

void cf2_set_trace(void* p) { g_cf2_trace = reinterpret_cast<long long*>(p); }

const Family kCf2Family = {cf2_validate, cf2_weight_count, cf2_weight_numel, cf2_packed_bytes,
                           cf2_pack,     cf2_ws,           cf2_forward,      cf2_init};

}  // namespace wl
