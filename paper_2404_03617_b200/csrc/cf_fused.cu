// cf_fused.cu — one-launch conv-first residual block on sm_100a.
//
// Covers the reference ConvFirst block (core.py:100-109; fused schedule
// machine.py:462-525) and the ConvNeXt-style variant (depthwise k x k,
// LayerNorm, GELU):
//     xc = conv_kxk_T(x) + b_conv [-> LayerNorm]
//     z  = x + b + sum_j phi(xc U_j + a_j) V_j        (loop fusion, Eq. ffn-eff)
// Only x and z cross HBM; the hidden activation lives in TMEM.
//
// Per persistent CTA, tiles of 16 x 8 output pixels (one tcgen05 M=128
// accumulator, M-block i = tile row i) flow through
//   producer warp : TMA 5-D halo load [G][TH+k-1][TW+k-1][8] (zero-filled
//                   padding), bulk copies of weight chunks [U_j | V_j]
//   MMA warp      : expand chunk j
//                   (SS: xc smem x U_j) -> TMEM E; project (TS: H in TMEM x
//                   V_j) accumulated into TMEM Z
//   H warps (4)   : E -> +a, phi -> fp16 -> TMEM H      (A operand of TS MMA)
//   T warps (4)   : the grouped T = 8 conv on the warp-level tensor path
//                   (mma.sync m16n8k16 / k8, K = 8 = T: ldmatrix fragments
//                   straight from the halo, weights as per-lane B fragments;
//                   round 1 ran it as block-diagonal M128 N16 tcgen05 MMAs,
//                   7/8 zeros) or the depthwise stencil on CUDA cores,
//                   LayerNorm, xc -> smem; final z = Z + b + x -> HBM
// Conv of tile t+1 is issued before the FFN of tile t so the T warps prepare
// the next tile while the tensor core runs the current one.
#include <cuda.h>
#include <cuda_fp16.h>
#include <cstdint>
#include "common.cuh"
#include "plan.h"

namespace wl {

struct CfArgs {
  CfPlan p;
  int n, h, w;
  int tiles_x, tiles_y, ntiles;
  float ln_eps;
  int norm;
  const uint8_t* wpack;
  __half* z;
  long long* trace;  // debug: clock64 stamps of CTA 0 (tools/trace_cf.py), null in production
};

namespace cfk {
constexpr int kThreads = 512;  // warps 12-15: second hidden-epilogue group (odd 16-column blocks)
constexpr int kProducerWarp = 0, kMmaWarp = 1, kAllocWarp = 2, kHWarp0 = 4, kTWarp0 = 8;

struct Bars {
  uint64_t hdr_full, w_all;
  uint64_t halo_full[8], halo_empty[8];
  uint64_t xc_full[2], xc_empty[2];
  uint64_t e_full[2], h_full[2], h_empty[2];
  uint64_t z_full, z_empty;
  uint64_t w_full[8], w_empty[8];
  uint32_t tmem_base;
};
}  // namespace cfk

#define CF_TRACE(it, k)                                                                 \
  do {                                                                                  \
    if (args.trace && blockIdx.x == 0 && (it) < 16) args.trace[8 + 12 * (it) + (k)] = clock64(); \
  } while (0)

template <int C, int KS, bool T8, int ACT>
__global__ void __launch_bounds__(cfk::kThreads, 2)
    cf_fused_kernel(const __grid_constant__ CUtensorMap tmap_x, const __grid_constant__ CfArgs args) {
  using namespace cfk;
  constexpr int G = C / 8;
  constexpr int P = KS / 2;
  constexpr int TH = 16, TW = 8;
  constexpr int HH = TH + KS - 1, HWD = TW + KS - 1;
  const CfPlan& pl = args.p;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* s_halo = smem + pl.s_halo;
  uint8_t* s_xc = smem + pl.s_xc;
  uint8_t* s_hdr = smem + pl.s_hdr;
  uint8_t* s_ring = smem + pl.s_ring;
  Bars& B = *reinterpret_cast<Bars*>(smem + pl.s_bar);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int r = pl.r, nchunks = pl.nchunks, S = pl.ring_stages, NHB = pl.halo_bufs;

  if (threadIdx.x == 0) {
    mbar_init(&B.hdr_full, 1);
    mbar_init(&B.w_all, 1);
    for (int i = 0; i < pl.halo_bufs; ++i) {
      mbar_init(&B.halo_full[i], 1);
      mbar_init(&B.halo_empty[i], 128);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&B.xc_full[i], 128);
      mbar_init(&B.xc_empty[i], 1);
      mbar_init(&B.e_full[i], 1);
      mbar_init(&B.h_full[i], 256);
      mbar_init(&B.h_empty[i], 1);
    }
    mbar_init(&B.z_full, 1);
    mbar_init(&B.z_empty, 128);
    for (int i = 0; i < S; ++i) {
      mbar_init(&B.w_full[i], 1);
      mbar_init(&B.w_empty[i], 1);
    }
    fence_mbar_init();
  }
  if (warp == kAllocWarp) tmem_alloc_n(&B.tmem_base, pl.tmem_cols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  pdl_trigger();  // single-wave persistent grid: let the next kernel stage its prologue
  pdl_wait();
  const uint32_t tmem = B.tmem_base;
  if (args.trace && blockIdx.x == 0 && threadIdx.x == 0) {
    args.trace[0] = clock64();
    args.trace[2] = pl.halo_bufs * 100 + nchunks;
    args.trace[3] = r;
  }

  const int tiles_per_img = args.tiles_x * args.tiles_y;
  auto tile_coords = [&](int t, int& n, int& y0, int& x0) {
    n = t / tiles_per_img;
    int rem = t % tiles_per_img;
    y0 = (rem / args.tiles_x) * TH;
    x0 = (rem % args.tiles_x) * TW;
  };
  const int my_tiles = (args.ntiles - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x;

  if (warp == kProducerWarp) {
    if (lane == 0) {
      prefetch_tmap(&tmap_x);
      mbar_arrive_expect_tx(&B.hdr_full, pl.hdr_bytes);
      bulk_g2s(s_hdr, args.wpack, pl.hdr_bytes, &B.hdr_full);
      const uint8_t* chunks = args.wpack + pl.hdr_bytes;
      if (pl.resident) {
        mbar_arrive_expect_tx(&B.w_all, nchunks * pl.chunk_bytes);
        for (int j = 0; j < nchunks; ++j)
          bulk_g2s(s_ring + j * pl.chunk_bytes, chunks + (size_t)j * pl.chunk_bytes, pl.chunk_bytes, &B.w_all);
      }
      auto load_halo = [&](int it) {
        int n, y0, x0;
        tile_coords((int)blockIdx.x + it * (int)gridDim.x, n, y0, x0);
        const int b = it % NHB, use = it / NHB;
        mbar_wait(&B.halo_empty[b], (use & 1) ^ 1);
        CF_TRACE(it, 0);
        mbar_arrive_expect_tx(&B.halo_full[b], pl.halo_bytes);
        tma_load_5d(s_halo + b * pl.halo_bytes, &tmap_x, 0, x0 - P, y0 - P, 0, n, &B.halo_full[b]);
      };
      for (int it = 0; it < my_tiles && it < NHB - 1; ++it) load_halo(it);
      for (int it = 0; it < my_tiles; ++it) {
        if (it + NHB - 1 < my_tiles) load_halo(it + NHB - 1);
        if (!pl.resident) {
          for (int j = 0; j < nchunks; ++j) {
            const int g = it * nchunks + j, slot = g % S, use = g / S;
            mbar_wait(&B.w_empty[slot], (use & 1) ^ 1);
            mbar_arrive_expect_tx(&B.w_full[slot], pl.chunk_bytes);
            bulk_g2s(s_ring + slot * pl.chunk_bytes, chunks + (size_t)j * pl.chunk_bytes, pl.chunk_bytes,
                     &B.w_full[slot]);
          }
        }
      }
    }
  } else if (warp == kMmaWarp) {
    {  // warp-converged issue: one elected lane issues each MMA / commit
      const uint32_t idesc_exp = make_idesc_f16(128, r);
      const uint32_t idesc_prj = make_idesc_f16(128, C);
      const uint32_t xc0 = smem_u32(s_xc), ring0 = smem_u32(s_ring);
      mbar_wait(&B.hdr_full, 0);
      if (pl.resident) mbar_wait(&B.w_all, 0);
      tc_fence_after();
      for (int it = 0; it < my_tiles; ++it) {
        const int xb = it & 1;
        mbar_wait(&B.xc_full[xb], (it >> 1) & 1);
        if (lane == 0) CF_TRACE(it, 5);
        tc_fence_after();
        const uint32_t xcb = xc0 + xb * pl.xc_bytes;
        auto slot_addr = [&](int j, int g) -> uint32_t {
          return pl.resident ? ring0 + j * pl.chunk_bytes : ring0 + (g % S) * pl.chunk_bytes;
        };
        auto issue_project = [&](int j) {
          const int g = it * nchunks + j, hb = g & 1;
          mbar_wait(&B.h_full[hb], (g >> 1) & 1);
          if (j == 0 && it > 0) mbar_wait(&B.z_empty, (it - 1) & 1);
          tc_fence_after();
          const uint32_t vbase = slot_addr(j, g) + pl.u_bytes;
#pragma unroll 1
          for (int kk = 0; kk < r / 16; ++kk) {
            const uint64_t bd = make_sdesc(vbase + kk * 2 * (C * 16), C * 16, 128);
            mma_ts_w(tmem + pl.t_z, tmem + pl.t_h + hb * pl.h_stride + kk * 8, bd, idesc_prj, (j > 0 || kk > 0));
          }
          mma_commit_w(&B.h_empty[hb]);
          if (!pl.resident) mma_commit_w(&B.w_empty[g % S]);
        };
        for (int j = 0; j < nchunks; ++j) {
          const int g = it * nchunks + j, eb = g & 1;
          if (!pl.resident) mbar_wait(&B.w_full[g % S], (g / S) & 1);
          tc_fence_after();
          const uint32_t ubase = slot_addr(j, g);
#pragma unroll 1
          for (int kk = 0; kk < C / 16; ++kk) {
            const uint64_t ad = make_sdesc(xcb + kk * 2 * 2048, 2048, 128);
            const uint64_t bd = make_sdesc(ubase + kk * 2 * (r * 16), r * 16, 128);
            mma_ss_w(tmem + pl.t_e + eb * r, ad, bd, idesc_exp, kk > 0);
          }
          mma_commit_w(&B.e_full[eb]);
          if (j == nchunks - 1) mma_commit_w(&B.xc_empty[xb]);
          if (j > 0) issue_project(j - 1);
        }
        issue_project(nchunks - 1);
        mma_commit_w(&B.z_full);
        if (lane == 0) CF_TRACE(it, 8);
      }
    }
  } else if ((warp >= kHWarp0 && warp < kHWarp0 + 4) || warp >= 12) {
    // ---------------- hidden epilogue: E -> +a, phi -> fp16 -> TMEM H
    // (two warp groups per TMEM quadrant, alternating 16-column blocks)
    const int q = warp % 4, hsub = warp >= 12 ? 1 : 0;
    const float* s_a = reinterpret_cast<const float*>(s_hdr + pl.o_a);
    mbar_wait(&B.hdr_full, 0);
    for (int it = 0; it < my_tiles; ++it) {
      for (int j = 0; j < nchunks; ++j) {
        const int g = it * nchunks + j, b = g & 1;
        mbar_wait(&B.e_full[b], (g >> 1) & 1);
        mbar_wait(&B.h_empty[b], ((g >> 1) & 1) ^ 1);
        if (q == 0 && lane == 0 && j == 0 && !hsub) CF_TRACE(it, 6);
        tc_fence_after();
        const float* aj = s_a + j * r;
#pragma unroll 1
        for (int c0 = hsub * 16; c0 < r; c0 += 32) {
          uint32_t v[16];
          WL_TMEM_LD16(tmem_lane_addr(tmem, q, pl.t_e + b * r + c0), v);
          tmem_ld_wait();
          uint4 o2[2];
          o2[0] = bias_act8<ACT>(v, aj + c0);
          o2[1] = bias_act8<ACT>(v + 8, aj + c0 + 8);
          const uint32_t* o = reinterpret_cast<const uint32_t*>(o2);
          WL_TMEM_ST8(tmem_lane_addr(tmem, q, pl.t_h + b * pl.h_stride + c0 / 2), o);
        }
        tmem_st_wait();
        tc_fence_before();
        mbar_arrive(&B.h_full[b]);
        if (q == 0 && lane == 0 && j == nchunks - 1 && !hsub) CF_TRACE(it, 7);
      }
    }
  } else if (warp >= kTWarp0 && warp < kTWarp0 + 4) {
    // ---------------- tile warps: conv epilogue / stencil, final epilogue
    const int q = warp - kTWarp0;
    const int m = q * 32 + lane;  // pixel of the tile == TMEM lane
    const int tr = m / 8, tc = m % 8;
    const float* s_bconv = reinterpret_cast<const float*>(s_hdr + pl.o_bconv);
    const float* s_lng = reinterpret_cast<const float*>(s_hdr + pl.o_lng);
    const float* s_lnb = reinterpret_cast<const float*>(s_hdr + pl.o_lnb);
    const float* s_b = reinterpret_cast<const float*>(s_hdr + pl.o_b);
    mbar_wait(&B.hdr_full, 0);

    auto conv_epi = [&](int u) {
      const int xb = u & 1;
      uint8_t* xcb = s_xc + xb * pl.xc_bytes;
      // LayerNorm statistics on values shifted by the pixel's first channel
      // (a sample of the same distribution): no E[x^2] - mean^2 cancellation
      // for large-mean activations
      float sum = 0.f, sq = 0.f, piv = 0.f;
      mbar_wait(&B.halo_full[u % NHB], (u / NHB) & 1);
      mbar_wait(&B.xc_empty[xb], ((u >> 1) & 1) ^ 1);
      if (q == 0 && lane == 0) CF_TRACE(u, 3);
      if constexpr (T8) {
        // warp q: fragments f = 2q, 2q + 1 (16 pixels = tile rows 2f, 2f + 1),
        // every group g: 4 k16 tap pairs + 1 k8 tap on mma.sync; lanes 0-15
        // address tap a of a pair, 16-31 tap b (the A fragment's K halves)
        const uint8_t* hb = s_halo + (u % NHB) * pl.halo_bytes;
        const uint32_t* frag = reinterpret_cast<const uint32_t*>(s_hdr + pl.o_convw);
        const int gid = lane >> 2, tq = lane & 3, lrow = lane & 15, lsel = lane >> 4;
        static constexpr int kTapA[4] = {0, 3, 6, 2}, kTapB[4] = {1, 4, 7, 5};
#pragma unroll 1
        for (int g = 0; g < G; ++g) {
          uint32_t bw[9];
#pragma unroll
          for (int i = 0; i < 9; ++i) bw[i] = frag[(g * 9 + i) * 32 + lane];
          const float2 bc = *reinterpret_cast<const float2*>(s_bconv + g * 8 + tq * 2);
          const uint32_t plane = smem_u32(hb + g * HH * HWD * 16);
#pragma unroll
          for (int fi = 0; fi < 2; ++fi) {
            const int f = 2 * q + fi;
            const int pr = 2 * f + (lrow >> 3), pc = lrow & 7;  // this lane's ldmatrix row: tile pixel
            float acc[4] = {bc.x, bc.y, bc.x, bc.y};
#pragma unroll
            for (int pp = 0; pp < 4; ++pp) {
              const int t = lsel ? kTapB[pp] : kTapA[pp];
              uint32_t a0, a1, a2, a3;
              ldsm_x4(plane + (uint32_t)(((pr + t / 3) * HWD + pc + t % 3) * 16), a0, a1, a2, a3);
              hmma16(acc, a0, a1, a2, a3, bw[2 * pp], bw[2 * pp + 1]);
            }
            {
              uint32_t a0, a1;
              ldsm_x2(plane + (uint32_t)(((pr + 2) * HWD + pc + 2) * 16), a0, a1);
              hmma8(acc, a0, a1, bw[8]);
            }
            const int m0 = 16 * f + gid;
            *reinterpret_cast<__half2*>(xcb + g * 2048 + m0 * 16 + tq * 4) = __floats2half2_rn(acc[0], acc[1]);
            *reinterpret_cast<__half2*>(xcb + g * 2048 + (m0 + 8) * 16 + tq * 4) = __floats2half2_rn(acc[2], acc[3]);
          }
        }
      } else {
        // depthwise k x k stencil on CUDA cores, fp32 accumulation
        const uint8_t* hb = s_halo + (u % NHB) * pl.halo_bytes;
        const float* s_w = reinterpret_cast<const float*>(s_hdr + pl.o_convw);  // [KS*KS][C]
#pragma unroll 1
        for (int g = 0; g < G; ++g) {
          float f[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) f[i] = s_bconv[g * 8 + i];
#pragma unroll 1
          for (int dy = 0; dy < KS; ++dy) {
#pragma unroll
            for (int dx = 0; dx < KS; ++dx) {
              const uint4 qv = lds128(hb + ((g * HH + tr + dy) * HWD + tc + dx) * 16);
              float hv[8];
              unpack8(qv, hv);
              const float4 w0 = *reinterpret_cast<const float4*>(s_w + (dy * KS + dx) * C + g * 8);
              const float4 w1 = *reinterpret_cast<const float4*>(s_w + (dy * KS + dx) * C + g * 8 + 4);
              f[0] += hv[0] * w0.x; f[1] += hv[1] * w0.y; f[2] += hv[2] * w0.z; f[3] += hv[3] * w0.w;
              f[4] += hv[4] * w1.x; f[5] += hv[5] * w1.y; f[6] += hv[6] * w1.z; f[7] += hv[7] * w1.w;
            }
          }
          if (g == 0) piv = f[0];
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const float dv = f[i] - piv;
            sum += dv;
            sq += dv * dv;
          }
          *reinterpret_cast<uint4*>(xcb + g * 2048 + m * 16) = pack8(f);
        }
      }
      if (args.norm) {
        // LayerNorm over the C channels of this pixel (biased variance)
        const float dm = sum * (1.f / C);
        const float mean = piv + dm;
        const float var = fmaxf(sq * (1.f / C) - dm * dm, 0.f);
        const float rstd = rsqrtf(var + args.ln_eps);
#pragma unroll 1
        for (int g = 0; g < G; ++g) {
          uint4* ptr = reinterpret_cast<uint4*>(xcb + g * 2048 + m * 16);
          float f[8];
          unpack8(*ptr, f);
#pragma unroll
          for (int i = 0; i < 8; ++i) f[i] = (f[i] - mean) * rstd * s_lng[g * 8 + i] + s_lnb[g * 8 + i];
          *ptr = pack8(f);
        }
      }
      fence_async_smem();
      mbar_arrive(&B.xc_full[xb]);
      if (q == 0 && lane == 0) CF_TRACE(u, 4);
    };

    auto final_epi = [&](int it) {
      int n, y0, x0;
      tile_coords((int)blockIdx.x + it * (int)gridDim.x, n, y0, x0);
      const int hbuf = it % NHB;
      mbar_wait(&B.z_full, it & 1);
      mbar_wait(&B.halo_full[hbuf], (it / NHB) & 1);
      if (q == 0 && lane == 0) CF_TRACE(it, 9);
      tc_fence_after();
      const uint8_t* hb = s_halo + hbuf * pl.halo_bytes;
      const int y = y0 + tr, x = x0 + tc;
      const bool inside = (y < args.h) && (x < args.w);
      __half* zp = args.z + (((size_t)n * args.h + y) * args.w + x) * C;
#pragma unroll 1
      for (int c0 = 0; c0 < C; c0 += 16) {
        uint32_t v[16];
        WL_TMEM_LD16(tmem_lane_addr(tmem, q, pl.t_z + c0), v);
        tmem_ld_wait();
        float f[16], res[16];
        unpack8(lds128(hb + (((c0 / 8) * HH + tr + P) * HWD + tc + P) * 16), res);
        unpack8(lds128(hb + (((c0 / 8 + 1) * HH + tr + P) * HWD + tc + P) * 16), res + 8);
        float b16[16];
        load16f(s_b + c0, b16);
#pragma unroll
        for (int i = 0; i < 16; ++i) f[i] = __uint_as_float(v[i]) + b16[i] + res[i];
        if (inside) {
          reinterpret_cast<uint4*>(zp + c0)[0] = pack8(f);
          reinterpret_cast<uint4*>(zp + c0)[1] = pack8(f + 8);
        }
      }
      tc_fence_before();
      mbar_arrive(&B.z_empty);
      mbar_arrive(&B.halo_empty[hbuf]);
      if (q == 0 && lane == 0) CF_TRACE(it, 10);
    };

    if (my_tiles > 0) conv_epi(0);
    for (int it = 0; it < my_tiles; ++it) {
      if (it + 1 < my_tiles) conv_epi(it + 1);
      final_epi(it);
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == kAllocWarp) tmem_dealloc_n(tmem, pl.tmem_cols);
}

}  // namespace wl

// =================================================================== host
#include <cstring>
#include <map>
#include <tuple>
#include "launch.h"

namespace wl {
long long* g_cf_trace = nullptr;
void cf_set_trace(void* p) { g_cf_trace = reinterpret_cast<long long*>(p); }

namespace {

constexpr int kSmemMax = 232448;          // 227 KB per CTA
constexpr int kSmemTwoPerSm = 112 * 1024;  // leaves room for 2 CTAs per SM

// plan with hidden chunks of r channels (0 when r does not fit TMEM)
bool cf_plan_r(const wl_block_desc& d, CfPlan& p, int r_want) {
  memset(&p, 0, sizeof(p));
  p.C = d.c;
  p.KS = d.ksize;
  p.T8 = d.group_width == 8 ? 1 : 0;
  p.hid = d.expansion * d.c;
  p.TH = 16;
  p.TW = 8;
  p.HH = p.TH + p.KS - 1;
  p.HW = p.TW + p.KS - 1;
  p.G = p.C / 8;
  const int zc = p.C, cc = 0;  // (the T = 8 conv no longer accumulates in TMEM)
  if (p.hid % r_want || zc + cc + 2 * r_want + 2 * align_up(r_want / 2, 16) > 512) return false;
  const int best = r_want;
  p.r = best;
  p.nchunks = p.hid / p.r;
  p.t_z = 0;
  p.t_cacc = zc;
  p.t_e = zc + cc;
  p.t_h = p.t_e + 2 * p.r;
  p.h_stride = align_up(p.r / 2, 16);
  const int cols = p.t_h + 2 * p.h_stride;
  p.tmem_cols = 32;
  while (p.tmem_cols < cols) p.tmem_cols *= 2;
  // header (fp32 vectors + conv weights)
  int o = 0;
  p.o_convw = o;
  o += p.T8 ? (p.C / 8) * 9 * 32 * 4 : p.KS * p.KS * p.C * 4;  // T8: per-lane mma.sync B fragments
  o = align_up(o, 16);
  p.o_bconv = o;
  o = align_up(o + p.C * 4, 16);
  p.o_lng = o;
  o = align_up(o + p.C * 4, 16);
  p.o_lnb = o;
  o = align_up(o + p.C * 4, 16);
  p.o_a = o;
  o = align_up(o + p.hid * 4, 16);
  p.o_b = o;
  o = align_up(o + p.C * 4, 16);
  p.hdr_bytes = o;
  p.u_bytes = p.r * p.C * 2;
  p.chunk_bytes = 2 * p.u_bytes;
  p.halo_bytes = p.G * p.HH * p.HW * 16;
  p.xc_bytes = kTileM * p.C * 2;
  p.s_halo = 0;
  const int all = p.nchunks * p.chunk_bytes;
  // deepest halo ring (4..2) that keeps two CTAs per SM; else one CTA per SM
  // with resident weights; else a streamed weight ring
  auto layout = [&](int nb) {
    p.halo_bufs = nb;
    p.s_xc = align_up(nb * p.halo_bytes, 128);
    p.s_hdr = p.s_xc + 2 * p.xc_bytes;
    p.s_ring = align_up(p.s_hdr + p.hdr_bytes, 128);
  };
  auto total = [&](int ring_bytes) { return align_up(p.s_ring + ring_bytes, 128) + 512; };
  bool placed = false;
  for (int nb = 8; nb >= 2 && !placed; --nb) {
    layout(nb);
    if (total(all) <= kSmemTwoPerSm && p.tmem_cols <= 256) {
      p.resident = 1;
      p.ctas_per_sm = 2;
      p.ring_stages = 1;
      placed = true;
    }
  }
  for (int nb = 8; nb >= 2 && !placed; --nb) {
    layout(nb);
    if (total(all) <= kSmemMax) {
      p.resident = 1;
      p.ctas_per_sm = 1;
      p.ring_stages = 1;
      placed = true;
    }
  }
  for (int nb = 8; nb >= 2 && !placed; --nb) {
    layout(nb);
    p.resident = 0;
    p.ctas_per_sm = 1;
    p.ring_stages = 0;
    for (int s = 8; s >= 2; --s)
      if (total(s * p.chunk_bytes) <= kSmemMax) {
        p.ring_stages = s;
        placed = true;
        break;
      }
  }
  if (!placed) return false;
  const int ring = p.resident ? all : p.ring_stages * p.chunk_bytes;
  p.s_bar = align_up(p.s_ring + ring, 128);
  p.smem_bytes = p.s_bar + 512;
  return true;
}

// Widest hidden chunk that still gives two CTAs per SM; else the widest that
// fits one CTA. (Narrow chunks only pay when they buy the second CTA: for wide
// blocks whose weights cannot fit twice, e.g. C = 96 x 6, a 16-wide chunk
// turned the FFN into 36 latency-bound N = 16 steps per tile — 76k cycles per
// tile at 56x56x96, measured.)
bool cf_plan(const wl_block_desc& d, CfPlan& p) {
  for (int r = 128; r >= 16; r -= 16)
    if (cf_plan_r(d, p, r) && p.ctas_per_sm == 2) return true;
  for (int r = 128; r >= 16; r -= 16)
    if (cf_plan_r(d, p, r)) return true;
  return false;
}

using CfKernel = void (*)(const CUtensorMap, const CfArgs);
using CfKey = std::tuple<int, int, int, int>;  // C, KS, T8, ACT

std::map<CfKey, CfKernel>& cf_table() {
  static std::map<CfKey, CfKernel> t;
  return t;
}

template <int C, int KS, bool T8>
void reg3() {
  cf_table()[CfKey{C, KS, T8, kRelu}] = cf_fused_kernel<C, KS, T8, kRelu>;
  cf_table()[CfKey{C, KS, T8, kSilu}] = cf_fused_kernel<C, KS, T8, kSilu>;
  cf_table()[CfKey{C, KS, T8, kGelu}] = cf_fused_kernel<C, KS, T8, kGelu>;
}
template <int C>
void reg_c() {
  reg3<C, 3, true>();
  reg3<C, 3, false>();
  reg3<C, 7, false>();
}
void cf_register() {
  static bool done = false;
  if (done) return;
  done = true;
  reg_c<16>();
  reg_c<32>();
  reg_c<48>();
  reg_c<64>();
  reg_c<80>();  // ConvFirstNet-Tiny's 72 channels, padded to a whole channel pair
  reg_c<96>();
  reg_c<128>();
}

int cf_validate(const wl_block_desc& d) {
  if (d.n < 1 || d.h < 1 || d.w < 1 || d.c < 1) return set_error(WL_EINVAL, "dims must be positive");
  if (d.expansion < 1) return set_error(WL_EINVAL, "expansion must be at least 1");
  if (d.group_width < 1 || d.c % d.group_width)
    return set_error(WL_EINVAL, "group width %d does not divide %d channels", d.group_width, d.c);
  if (d.stride != 1 && d.stride != 2) return set_error(WL_EINVAL, "stride must be 1 or 2");
  if (d.stride == 1 && d.k != d.c) return set_error(WL_EINVAL, "stride-1 blocks keep their channel count");
  if (d.ksize % 2 == 0 || d.ksize < 1) return set_error(WL_EINVAL, "conv kernel must be odd");
  if (d.norm != WL_NORM_NONE && d.norm != WL_NORM_LAYERNORM) return set_error(WL_EINVAL, "unknown norm");
  if (d.act < 0 || d.act > 4) return set_error(WL_EINVAL, "unknown activation");
  if (d.stride == 2) return kCf2Family.validate(d);
  if (cnx_wide(d)) return cnx_wide_validate(d);
  if (cf_wide(d)) return cf_wide_validate(d);
  if (d.act != kRelu && d.act != kSilu && d.act != kGelu)
    return set_error(WL_EUNSUPPORTED, "fused conv-first block supports relu/silu/gelu");
  const bool t8 = d.group_width == 8 && d.ksize == 3 && d.norm == WL_NORM_NONE;
  const bool t1 = d.group_width == 1 && (d.ksize == 3 || d.ksize == 7);
  if (!t8 && !t1)
    return set_error(WL_EUNSUPPORTED, "fused conv-first block supports T=8 3x3 or depthwise 3x3/7x7 (got T=%d k=%d)",
                     d.group_width, d.ksize);
  cf_register();
  if (!cf_table().count(CfKey{d.c, d.ksize, t8 ? 1 : 0, d.act}))
    return set_error(WL_EUNSUPPORTED, "no fused kernel instantiated for C=%d", d.c);
  CfPlan p;
  if (!cf_plan(d, p)) return set_error(WL_EUNSUPPORTED, "no launch plan fits C=%d hidden=%d", d.c, d.c * d.expansion);
  return WL_OK;
}

int cf_weight_count(const wl_block_desc& d) {
  if (d.stride == 2) return kCf2Family.weight_count(d);
  return d.norm == WL_NORM_LAYERNORM ? 8 : 6;
}

int64_t cf_weight_numel(const wl_block_desc& d, int i) {
  if (d.stride == 2) return kCf2Family.weight_numel(d, i);
  const int64_t c = d.c, hid = (int64_t)d.expansion * d.c;
  // [w_conv (C,k,k,T), b_conv (C), (ln_gamma, ln_beta), u (C,hid), a (hid), v (hid,C), b (C)]
  const bool ln = d.norm == WL_NORM_LAYERNORM;
  if (i == 0) return c * d.ksize * d.ksize * d.group_width;
  if (i == 1) return c;
  if (ln && (i == 2 || i == 3)) return c;
  const int j = ln ? i - 2 : i;
  switch (j) {
    case 2: return c * hid;
    case 3: return hid;
    case 4: return hid * c;
    case 5: return c;
  }
  return set_error(WL_EINVAL, "weight index %d out of range", i);
}

int64_t cf_packed_bytes(const wl_block_desc& d) {
  if (d.stride == 2) return kCf2Family.packed_bytes(d);
  if (cnx_wide(d)) return cnx_wide_pb(d);
  if (cf_wide(d)) return cf_wide_pb(d);
  CfPlan p;
  cf_plan(d, p);
  return (int64_t)p.hdr_bytes + (int64_t)p.nchunks * p.chunk_bytes;
}

int cf_pack(const wl_block_desc& d, const float* const* w, uint8_t* out) {
  if (d.stride == 2) return kCf2Family.pack(d, w, out);
  if (cnx_wide(d)) return cnx_wide_pack(d, w, out);
  if (cf_wide(d)) return cf_wide_pack(d, w, out);
  CfPlan p;
  cf_plan(d, p);
  memset(out, 0, (size_t)cf_packed_bytes(d));
  const bool ln = d.norm == WL_NORM_LAYERNORM;
  const float *wc = w[0], *bc = w[1];
  const float* lng = ln ? w[2] : nullptr;
  const float* lnb = ln ? w[3] : nullptr;
  const int o = ln ? 4 : 2;
  const float *u = w[o], *a = w[o + 1], *v = w[o + 2], *b = w[o + 3];
  const int C = p.C, KS = p.KS, hid = p.hid, r = p.r;
  uint8_t* hdr = out;
  if (p.T8) {
    // mma.sync B fragments [group][slot][lane] = (w[co][tap][ci], w[co][tap][ci + 1]),
    // co = 8 g + lane / 4, ci = 2 (lane % 4); slots hold the taps in k16-pair
    // order (0,1) (3,4) (6,7) (2,5) 8 (w_conv is (C, 3, 3, T = 8))
    static const int kTapOfSlot[9] = {0, 1, 3, 4, 6, 7, 2, 5, 8};
    for (int g = 0; g < C / 8; ++g)
      for (int slot = 0; slot < 9; ++slot)
        for (int l = 0; l < 32; ++l) {
          const int tap = kTapOfSlot[slot], co = 8 * g + l / 4, ci = 2 * (l % 4);
          const size_t off = (size_t)p.o_convw + (((size_t)g * 9 + slot) * 32 + l) * 4;
          put_h(hdr, off, wc[((size_t)co * 9 + tap) * 8 + ci]);
          put_h(hdr, off + 2, wc[((size_t)co * 9 + tap) * 8 + ci + 1]);
        }
  } else {
    float* cw = reinterpret_cast<float*>(hdr + p.o_convw);
    for (int ch = 0; ch < C; ++ch)
      for (int t = 0; t < KS * KS; ++t) cw[t * C + ch] = wc[(size_t)ch * KS * KS + t];
  }
  float* fb = reinterpret_cast<float*>(hdr + p.o_bconv);
  float* fg = reinterpret_cast<float*>(hdr + p.o_lng);
  float* fbt = reinterpret_cast<float*>(hdr + p.o_lnb);
  float* fa = reinterpret_cast<float*>(hdr + p.o_a);
  float* fbb = reinterpret_cast<float*>(hdr + p.o_b);
  for (int ch = 0; ch < C; ++ch) {
    fb[ch] = bc[ch];
    fg[ch] = ln ? lng[ch] : 1.f;
    fbt[ch] = ln ? lnb[ch] : 0.f;
    fbb[ch] = b[ch];
  }
  for (int i = 0; i < hid; ++i) fa[i] = a[i];
  for (int j = 0; j < p.nchunks; ++j) {
    uint8_t* ch = out + p.hdr_bytes + (size_t)j * p.chunk_bytes;
    for (int n = 0; n < r; ++n)
      for (int k = 0; k < C; ++k) put_h(ch, core_off_h(n, k, r * 16), u[(size_t)k * hid + j * r + n]);
    uint8_t* vch = ch + p.u_bytes;
    for (int n = 0; n < C; ++n)
      for (int k = 0; k < r; ++k) put_h(vch, core_off_h(n, k, C * 16), v[(size_t)(j * r + k) * C + n]);
  }
  return WL_OK;
}

int64_t cf_workspace(const wl_block_desc& d) {
  if (d.stride == 2) return kCf2Family.workspace_bytes(d);
  if (cnx_wide(d)) return cnx_wide_ws(d);
  if (cf_wide(d)) return cf_wide_ws(d);
  return 0;
}

int cf_forward(const wl_block_desc& d, const void* x, const void* packed, void* z, void* ws, cudaStream_t st) {
  if (d.stride == 2) return kCf2Family.forward(d, x, packed, z, ws, st);
  if (cnx_wide(d)) return cnx_wide_fwd(d, x, packed, z, ws, st);
  if (cf_wide(d)) return cf_wide_fwd(d, x, packed, z, ws, st);
  CfPlan p;
  cf_plan(d, p);
  cf_register();
  const bool t8 = d.group_width == 8;
  auto it = cf_table().find(CfKey{d.c, d.ksize, t8 ? 1 : 0, d.act});
  if (it == cf_table().end()) return set_error(WL_EUNSUPPORTED, "kernel not instantiated");
  CUtensorMap tm;
  const uint64_t dims[5] = {8, (uint64_t)d.w, (uint64_t)d.h, (uint64_t)(d.c / 8), (uint64_t)d.n};
  const uint64_t strides[4] = {(uint64_t)d.c * 2, (uint64_t)d.w * d.c * 2, 16, (uint64_t)d.h * d.w * d.c * 2};
  const uint32_t box[5] = {8, (uint32_t)p.HW, (uint32_t)p.HH, (uint32_t)p.G, 1};
  if (int e = encode_tmap(&tm, x, 5, dims, strides, box)) return e;
  CfArgs a;
  a.p = p;
  a.n = d.n;
  a.h = d.h;
  a.w = d.w;
  a.tiles_x = (d.w + p.TW - 1) / p.TW;
  a.tiles_y = (d.h + p.TH - 1) / p.TH;
  a.ntiles = d.n * a.tiles_x * a.tiles_y;
  a.ln_eps = d.ln_eps > 0 ? d.ln_eps : 1e-6f;
  a.norm = d.norm;
  a.wpack = reinterpret_cast<const uint8_t*>(packed);
  a.z = reinterpret_cast<__half*>(z);
  a.trace = g_cf_trace;
  const int grid = std::min(a.ntiles, kNumSMs * p.ctas_per_sm);
  return launch_pdl(it->second, grid, cfk::kThreads, p.smem_bytes, st, "cf_fused launch", tm, a);
}

int cf_init() {
  cf_register();
  for (auto& kv : cf_table())
    if (int e = check_cuda(cudaFuncSetAttribute(kv.second, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemMax),
                           "cudaFuncSetAttribute(cf)"))
      return e;
  return WL_OK;
}

}  // namespace

const Family kCfFamily = {cf_validate, cf_weight_count, cf_weight_numel, cf_packed_bytes,
                          cf_pack,     cf_workspace,    cf_forward,      cf_init};

}  // namespace wl
