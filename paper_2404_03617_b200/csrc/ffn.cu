// ffn.cu — fused FFN z = phi(x U + a) V + b (+ res) with the expanded hidden
// kept on chip: the FFN block (core.py:125-132; the fused schedule's chunk
// identity, machine.py:236-252 / PAPER.md:862-866) and the pointwise half of
// the wide ConvNeXt blocks (C = 192 / 256 / 384; cnx.cu computes the
// depthwise conv + LayerNorm that produces x).
//
// Per CTA, persistent over 128-row tiles:
//   A = x tile (128 x C) in shared memory, 128B-swizzled slabs of 64 channels
//   for each hidden chunk j of HC channels:
//     E_j  = A . U_j              tcgen05 SS -> TMEM (double-buffered)
//     H_j  = phi(E_j + a_j)       8 epilogue warps, packed fp16 written back
//                                 IN PLACE over E_j's columns (tcgen05.st)
//     Z   += H_j . V_j            tcgen05 TS (A operand from TMEM)
//   z = Z + b (+ res)             staged in the A buffer, TMA-stored
// TMEM: Z (C columns) + 2 x HC (E/H) <= 512: HC = 128 for C <= 256, 64 for
// C <= 384. U_j / V_j stream through a ring of shared-memory stages (TMA,
// 128B swizzle) in the order U0 V0 U1 V1 ..., consumed E0 E1 P0 E2 P1 ...
// Only x, the weights (L2-resident across tiles) and z cross HBM.
#include <cuda.h>
#include <cuda_fp16.h>
#include <cstdint>
#include <algorithm>
#include <cstring>
#include "common.cuh"
#include "launch.h"
#include "plan.h"

namespace wl {

namespace ff {
constexpr int kEpiWarps = 8;  // kGroups warp groups per TMEM lane quadrant
constexpr int kGroups = kEpiWarps / 4;
constexpr int kHU = 128 / kGroups / 16;  // 16-column units of E per warp (HC <= 128)
constexpr int kXWarp = 2 + kEpiWarps;
constexpr int kVWarp = kXWarp + 1;
constexpr int kThreads = (kVWarp + 1) * 32;  // warp 0 U-slab loads, 1 MMA, epilogue, x / residual TMA, V-slab loads
constexpr int kMaxStages = 6;
constexpr int kSmemMax = 232448;
struct Args {
  int M, C, hid, HC, nch, act, has_res;
  int tiles, slabs, stage_bytes, stages, s_ring, u_bytes, v_bytes;
  int NU, NV, us_bytes, vs_bytes, s_vring;  // U-slab / V-slab rings: stage counts, slab bytes, V ring offset
  const uint8_t* wimg;  // per hidden chunk: [U_j image][V_j image] (ffn_pack_images)
  int resident;  // all 2 nch weight stages fit: loaded once, never recycled
  int NA;        // x tile buffers (2: the next tile's x loads while this one computes)
  int direct;    // NA == 1: z leaves by direct stores (res read from global), x is freed at the last expansion
  const __half* res;
  __half* z;
  long long* trace;  // debug: CTA 0 clock64 stamps (wl_debug_set_trace)
  int t_z, t_e;  // TMEM column bases
  int NE;        // E / H buffers in TMEM (3 when C + 3 HC fits: the next-but-one expansion need not wait for a projection)
  uint32_t tmem_cols;
  const float* a;  // hidden bias [hid]
  const float* b;  // output bias [C]
};
struct Bars {
  uint64_t a_full[2], a_free[2], a_used[2], res_full[2];
  uint64_t u_full[16], u_empty[16], v_full[16], v_empty[16];
  uint64_t e_full[3], h_full[3], p_done[3];
  uint64_t z_full, z_empty;
  uint32_t tmem_base;
};
}  // namespace ff

__device__ __forceinline__ void ff_tma2(void* dst, const void* tmap, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
      "[%4];" ::"r"(smem_u32(dst)),
      "l"(tmap), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void ff_store2(const void* tmap, const void* src, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(tmap),
               "r"(smem_u32(src)), "r"(c0), "r"(c1)
               : "memory");
}
#define FF_TRACE(slot)                                                              \
  do {                                                                              \
    if (a.trace && blockIdx.x == 0 && (slot) < 4096) a.trace[(slot)] = clock64();   \
  } while (0)
// 1-D bulk copy with an L2 evict_last hint: the weight images are re-read by
// every tile of every CTA and should outlive the streamed activations in L2
__device__ __forceinline__ void bulk_g2s_keep(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                              uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void ff_bar(int n) { asm volatile("bar.sync 2, %0;" ::"r"(n) : "memory"); }

template <int ACT, typename T>
__global__ void __launch_bounds__(ff::kThreads, 1)
    ffn_fused_kernel(const __grid_constant__ CUtensorMap tx, const __grid_constant__ CUtensorMap tu,
                     const __grid_constant__ CUtensorMap tv, const __grid_constant__ CUtensorMap tr,
                     const __grid_constant__ CUtensorMap tz, const __grid_constant__ ff::Args a) {
  using namespace ff;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* s_a = smem;  // A tile; later the residual / output staging
  uint8_t* s_ring = smem + a.s_ring;
  uint8_t* s_vring = smem + a.s_vring;
  Bars& B = *reinterpret_cast<Bars*>(s_vring + a.NV * a.vs_bytes);
  float* s_abias = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(&B) + ((sizeof(Bars) + 15) / 16) * 16);
  float* s_bbias = s_abias + a.hid;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int C = a.C, HC = a.HC, nch = a.nch;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 2; ++i) {
      mbar_init(&B.a_full[i], 1);
      mbar_init(&B.a_free[i], 1);
      mbar_init(&B.a_used[i], 1);
      mbar_init(&B.res_full[i], 1);
    }
    for (int s = 0; s < a.NU; ++s) {
      mbar_init(&B.u_full[s], 1);  // (resident: one phase, never recycled)
      mbar_init(&B.u_empty[s], 1);
    }
    for (int s = 0; s < a.NV; ++s) {
      mbar_init(&B.v_full[s], 1);
      mbar_init(&B.v_empty[s], 1);
    }
    for (int i = 0; i < 3; ++i) {
      mbar_init(&B.e_full[i], 1);
      mbar_init(&B.h_full[i], kEpiWarps);
      mbar_init(&B.p_done[i], 1);
    }
    mbar_init(&B.z_full, 1);
    mbar_init(&B.z_empty, kEpiWarps);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc_n(&B.tmem_base, a.tmem_cols);
  for (int i = threadIdx.x; i < a.hid; i += blockDim.x) s_abias[i] = a.a[i];
  for (int i = threadIdx.x; i < a.C; i += blockDim.x) s_bbias[i] = a.b[i];
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  pdl_trigger();
  pdl_wait();
  const uint32_t tmem = B.tmem_base;
  if (threadIdx.x == 0) FF_TRACE(15);
  const int my_tiles = blockIdx.x < a.tiles ? (a.tiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const int per_tile = 2 * nch;  // weight stages per tile
  // each CTA walks the hidden chunks from its own starting offset, so the 148
  // CTAs' weight reads spread over all of U / V instead of converging on the
  // same few L2 lines (the Z sum is order-independent up to fp32 rounding)
  const int rot = 0;  // (a per-CTA rotation of the chunk order measured slower: 141 -> 152 us at C = 192)

  if (warp == 0 || warp == kVWarp) {
    if (lane == 0) {
      // ----------------------------------------------------- weight producers
      prefetch_tmap(&tx);
      prefetch_tmap(&tu);
      prefetch_tmap(&tv);
      uint64_t keep;
      asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(keep));
      // U_j / V_j arrive as pre-swizzled shared-memory images (packed on the
      // host), one 1-D bulk copy per K-slab, into two rings (U slabs, V slabs)
      // in the order the MMA consumes them: E0 E1 P0 E2 P1 ... P(n-1)
      const int uslabs = a.slabs, vslabs = HC / 64;
      int useq = 0, vseq = 0;
      auto load_u = [&](int j) {
        for (int sl = 0; sl < uslabs; ++sl, ++useq) {
          const int s = useq % a.NU;
          if (!a.resident) mbar_wait(&B.u_empty[s], ((useq / a.NU) & 1) ^ 1);
          mbar_arrive_expect_tx(&B.u_full[s], a.us_bytes);
          bulk_g2s_keep(s_ring + s * a.us_bytes, a.wimg + (size_t)j * (a.u_bytes + a.v_bytes) + sl * a.us_bytes,
                        a.us_bytes, &B.u_full[s], keep);
        }
      };
      auto load_v = [&](int j) {
        for (int sl = 0; sl < vslabs; ++sl, ++vseq) {
          const int s = vseq % a.NV;
          if (!a.resident) mbar_wait(&B.v_empty[s], ((vseq / a.NV) & 1) ^ 1);
          mbar_arrive_expect_tx(&B.v_full[s], a.vs_bytes);
          bulk_g2s_keep(s_vring + s * a.vs_bytes,
                        a.wimg + (size_t)j * (a.u_bytes + a.v_bytes) + a.u_bytes + sl * a.vs_bytes, a.vs_bytes,
                        &B.v_full[s], keep);
        }
      };
      // the U and V rings are filled by two threads (warp 0 lane 0: U, lane 0 of
      // kVWarp: V) so a wait on one ring never holds back the other
      const bool vthread = warp == kVWarp;
      for (int t = 0; t < (a.resident ? (my_tiles > 0 ? 1 : 0) : my_tiles); ++t)
        for (int j = 0; j < nch; ++j) {
          if (vthread)
            load_v(j);
          else
            load_u(j);
        }
    }
  } else if (warp == kXWarp) {
    if (lane == 0) {
      // ----------------------------------------------- x / residual producer
      auto load_x = [&](int t) {
        const int b = t % a.NA, tile = blockIdx.x + t * gridDim.x;
        mbar_wait(&B.a_free[b], ((t / a.NA) & 1) ^ 1);
        mbar_arrive_expect_tx(&B.a_full[b], a.slabs * 16384);
        for (int sl = 0; sl < a.slabs; ++sl)
          ff_tma2(s_a + (b * a.slabs + sl) * 16384, &tx, sl * 64, tile * 128, &B.a_full[b]);
      };
      if (my_tiles > 0) load_x(0);
      for (int t = 0; t < my_tiles; ++t) {
        if (t + 1 < my_tiles) load_x(t + 1);
        if (a.has_res && !a.direct) {
          const int b = t % a.NA, tile = blockIdx.x + t * gridDim.x;
          mbar_wait(&B.a_used[b], (t / a.NA) & 1);  // the tile's last expansion has read x
          mbar_arrive_expect_tx(&B.res_full[b], a.slabs * 16384);
          for (int sl = 0; sl < a.slabs; ++sl)
            ff_tma2(s_a + (b * a.slabs + sl) * 16384, &tr, sl * 64, tile * 128, &B.res_full[b]);
        }
      }
    }
  } else if (warp == 1) {
    {
      // ---------------------------------------------------------- MMA issuer
      // (the whole warp runs the loop; one elected lane issues each MMA / commit)
      const uint32_t idesc_e = make_idesc_f16(128, HC) | Dt<T>::kIdescAB;
      const int zn = C > 256 ? C / 2 : C;
      const uint32_t idesc_z = make_idesc_f16(128, zn) | Dt<T>::kIdescAB;
      const uint32_t sa = smem_u32(s_a), sr = smem_u32(s_ring), svr = smem_u32(s_vring);
      // ring positions of the streamed U / V slabs (incremental: an integer
      // division here is a MUFU.RCP queued behind the epilogue's GELU tanh)
      int us = 0, uph = 0, vs = 0, vph = 0;
      // The issue loop is latency-bound in this one thread (each tcgen05.mma
      // waits on its descriptor chain), so everything that does not change per
      // MMA is hoisted: descriptor bases advance by (byte offset >> 4) in their
      // start-address field, the TMEM A offsets of the projection's K steps are
      // a table, and resident weight stages are waited on once.
      const uint64_t du0 = make_sdesc_sw128(sr), dv0 = make_sdesc_sw128(svr);
      uint32_t aoff[8];  // K step kk of H_j: epilogue group hs packs its HC / G hidden at the start of its range
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        const int hs = (kk * 16) / (HC / kGroups), loc = kk * 16 - hs * (HC / kGroups);
        aoff[kk] = hs * (HC / kGroups) + loc / 2;
      }
      const int NE = a.NE, nsl = HC / 64, nr0 = C > 256 ? 2 : 1;
      int eb = 0, eph = 0;  // E buffer of the next expansion and its reuse count
      int pb = 0, pph = 0;  // E/H buffer of the next projection
      int xb = 0, xph = 0;
      for (int t = 0; t < my_tiles; ++t) {
        mbar_wait(&B.a_full[xb], xph & 1);
        tc_fence_after();
        const uint64_t dx0 = make_sdesc_sw128(sa + xb * a.slabs * 16384);
        const bool wait_w = !a.resident || t == 0;
        auto expand = [&](int j) {
          const int g = t * nch + j, b = eb;
          if (eph > 0) mbar_wait(&B.p_done[b], (eph - 1) & 1);  // H of this buffer's previous use consumed
          if (++eb == NE) eb = 0, ++eph;
          if (lane == 0) FF_TRACE(16 + g * 4 + 0);
          const uint32_t d = tmem + a.t_e + b * HC;
          for (int sl = 0; sl < a.slabs; ++sl) {
            const int s = a.resident ? (j * a.slabs + sl) : us;
            if (wait_w) {
              mbar_wait(&B.u_full[s], a.resident ? 0 : uph);
              tc_fence_after();
            }
            if (!a.resident && ++us == a.NU) us = 0, uph ^= 1;
            const uint64_t ad = dx0 + (uint64_t)(sl * (16384 >> 4)), bd = du0 + (uint64_t)(s * (a.us_bytes >> 4));
            const int nk = min(4, (C - sl * 64) / 16);  // zero-padded channels of a partial slab
#pragma unroll
            for (int k4 = 0; k4 < 4; ++k4)
              if (k4 < nk) mma_ss_w(d, ad + 2 * k4, bd + 2 * k4, idesc_e, (sl | k4) != 0);
            if (!a.resident) mma_commit_w(&B.u_empty[s]);
          }
          if (lane == 0) FF_TRACE(2000 + g * 2 + 0);
          mma_commit_w(&B.e_full[b]);
          if (j == nch - 1) mma_commit_w(a.direct ? &B.a_free[xb] : &B.a_used[xb]);
        };
        auto project = [&](int j) {
          const int g = t * nch + j, b = pb;
          mbar_wait(&B.h_full[b], pph & 1);
          if (++pb == NE) pb = 0, ++pph;
          if (j == 0 && t > 0) mbar_wait(&B.z_empty, (t - 1) & 1);
          if (lane == 0) FF_TRACE(16 + g * 4 + 1);
          const uint32_t ab = tmem + a.t_e + b * HC;
#pragma unroll
          for (int sl = 0; sl < 2; ++sl) {
            if (sl >= nsl) break;
            const int s = a.resident ? (j * nsl + sl) : vs;
            if (wait_w) {
              mbar_wait(&B.v_full[s], a.resident ? 0 : vph);
              tc_fence_after();
            }
            if (!a.resident && ++vs == a.NV) vs = 0, vph ^= 1;
            const uint64_t bd = dv0 + (uint64_t)(s * (a.vs_bytes >> 4));
            if (nr0 == 1) {
#pragma unroll
              for (int k4 = 0; k4 < 4; ++k4)
                mma_ts_w(tmem + a.t_z, ab + aoff[sl * 4 + k4], bd + 2 * k4, idesc_z, (j > 0 || sl > 0 || k4 > 0));
            } else {
#pragma unroll
              for (int k4 = 0; k4 < 4; ++k4)
#pragma unroll
                for (int r = 0; r < 2; ++r)
                  mma_ts_w(tmem + a.t_z + r * zn, ab + aoff[sl * 4 + k4], bd + (uint64_t)(r * zn * (128 >> 4)) + 2 * k4,
                         idesc_z, (j > 0 || sl > 0 || k4 > 0));
            }
            if (!a.resident) mma_commit_w(&B.v_empty[s]);
          }
          if (lane == 0) FF_TRACE(2000 + g * 2 + 1);
          mma_commit_w(&B.p_done[b]);
          if (j == nch - 1) mma_commit_w(&B.z_full);
        };
        for (int j = 0; j < nch && j < a.NE; ++j) expand(j);
        for (int j = 0; j < nch; ++j) {
          project(j);
          if (j + a.NE < nch) expand(j + a.NE);
        }
        if (++xb == a.NA) xb = 0, ++xph;
      }
    }
  } else {
    // ------------------------------------------------------------- epilogue
    const int q = warp & 3, grp = (warp - 2) >> 2;
    const int r = q * 32 + lane;
    const bool leader = threadIdx.x == 64;
    const int hw = HC / kGroups;  // hidden columns per warp group
    for (int t = 0; t < my_tiles; ++t) {
      const int tile = blockIdx.x + t * gridDim.x;
      for (int j = 0; j < nch; ++j) {
        const int g = t * nch + j, b = g % a.NE;
        const float* aj = s_abias + ((j + rot) % nch) * HC + grp * hw;
        mbar_wait(&B.e_full[b], (g / a.NE) & 1);
        tc_fence_after();
        if (threadIdx.x == 64) FF_TRACE(16 + g * 4 + 2);
        const uint32_t eb = tmem_lane_addr(tmem, q, a.t_e + b * HC + grp * hw);
        uint32_t v[16 * kHU];
#pragma unroll
        for (int u = 0; u < kHU; ++u)
          if (u * 16 < hw) WL_TMEM_LD16(eb + u * 16, (v + 16 * u));
        tmem_ld_wait();
#pragma unroll
        for (int u = 0; u < kHU; ++u)
          if (u * 16 < hw) {
            float bb[16];
            load16f(aj + u * 16, bb);
            uint32_t o[8];
#pragma unroll
            for (int i = 0; i < 8; ++i)
              o[i] = act_pack2<T, ACT>(__uint_as_float(v[16 * u + 2 * i]) + bb[2 * i],
                                       __uint_as_float(v[16 * u + 2 * i + 1]) + bb[2 * i + 1]);
            WL_TMEM_ST8(eb + u * 8, o);
          }
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&B.h_full[b]);
        if (threadIdx.x == 64) FF_TRACE(16 + g * 4 + 3);
      }
      // --------------------------------------------- z = Z + b (+ res)
      const int xb = t % a.NA;
      uint8_t* s_x = s_a + xb * a.slabs * 16384;
      const int units = C / 16, u_lo = grp * units / kGroups, u_hi = (grp + 1) * units / kGroups;
      const int64_t grow = (int64_t)tile * 128 + r;
      // direct stores: the residual rows are fetched from global before the wait
      // for Z, so their latency hides under the tile's last projection
      constexpr int kPre = 3;
      const bool pre = a.direct && a.has_res && u_hi - u_lo <= kPre;
      uint4 rpre[kPre][2];
      if (pre) {
#pragma unroll
        for (int i = 0; i < kPre; ++i)
#pragma unroll
          for (int hh = 0; hh < 2; ++hh)
            rpre[i][hh] = (u_lo + i < u_hi && grow < a.M)
                              ? __ldg(reinterpret_cast<const uint4*>(a.res + grow * C + (u_lo + i) * 16 + 8 * hh))
                              : make_uint4(0, 0, 0, 0);
      }
      mbar_wait(&B.z_full, t & 1);
      if (threadIdx.x == 64) FF_TRACE(3000 + 2 * t + 0);
      if (a.has_res && !a.direct) mbar_wait(&B.res_full[xb], (t / a.NA) & 1);
      tc_fence_after();
      const uint32_t zb = tmem_lane_addr(tmem, q, a.t_z);
      if (pre) {
#pragma unroll
        for (int i0 = 0; i0 < kPre; i0 += 2) {
          if (u_lo + i0 >= u_hi) break;
          uint32_t v[32];
#pragma unroll
          for (int jj = 0; jj < 2; ++jj)
            if (i0 + jj < kPre && u_lo + i0 + jj < u_hi) WL_TMEM_LD16(zb + (u_lo + i0 + jj) * 16, (v + 16 * jj));
          tmem_ld_wait();
#pragma unroll
          for (int jj = 0; jj < 2; ++jj)
            if (i0 + jj < kPre && u_lo + i0 + jj < u_hi && grow < a.M) {
              const int c16 = (u_lo + i0 + jj) * 16;
              float bb[16];
              load16f(s_bbias + c16, bb);
#pragma unroll
              for (int hh = 0; hh < 2; ++hh) {
                float f[8], rr[8];
                unpack8t<T>(rpre[i0 + jj][hh], rr);
#pragma unroll
                for (int i = 0; i < 8; ++i) f[i] = __uint_as_float(v[16 * jj + 8 * hh + i]) + bb[8 * hh + i] + rr[i];
                *reinterpret_cast<uint4*>(a.z + grow * C + c16 + 8 * hh) = pack8t<T>(f);
              }
            }
        }
      }
      for (int u0 = pre ? u_hi : u_lo; u0 < u_hi; u0 += 2) {
        uint32_t v[32];
#pragma unroll
        for (int jj = 0; jj < 2; ++jj)
          if (u0 + jj < u_hi) WL_TMEM_LD16(zb + (u0 + jj) * 16, (v + 16 * jj));
        tmem_ld_wait();
#pragma unroll
        for (int jj = 0; jj < 2; ++jj)
          if (u0 + jj < u_hi) {
            const int c16 = (u0 + jj) * 16, sl = c16 >> 6, c8 = (c16 & 63) >> 3;
            float bb[16];
            load16f(s_bbias + c16, bb);
            uint8_t* rowp = s_x + sl * 16384 + r * 128;
#pragma unroll
            for (int hh = 0; hh < 2; ++hh) {
              float f[8];
#pragma unroll
              for (int i = 0; i < 8; ++i) f[i] = __uint_as_float(v[16 * jj + 8 * hh + i]) + bb[8 * hh + i];
              if (a.direct) {
                if (grow < a.M) {
                  if (a.has_res) {
                    float rr[8];
                    unpack8t<T>(__ldg(reinterpret_cast<const uint4*>(a.res + grow * C + c16 + 8 * hh)), rr);
#pragma unroll
                    for (int i = 0; i < 8; ++i) f[i] += rr[i];
                  }
                  *reinterpret_cast<uint4*>(a.z + grow * C + c16 + 8 * hh) = pack8t<T>(f);
                }
              } else {
                uint8_t* p = rowp + (((c8 + hh) ^ (r & 7)) << 4);
                if (a.has_res) {
                  float rr[8];
                  unpack8t<T>(lds128(p), rr);
#pragma unroll
                  for (int i = 0; i < 8; ++i) f[i] += rr[i];
                }
                *reinterpret_cast<uint4*>(p) = pack8t<T>(f);
              }
            }
          }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&B.z_empty);
      if (threadIdx.x == 64) FF_TRACE(3000 + 2 * t + 1);
      if (!a.direct) {
        fence_async_smem();
        ff_bar(kEpiWarps * 32);
        if (leader) {
          for (int sl = 0; sl < a.slabs; ++sl) ff_store2(&tz, s_x + sl * 16384, sl * 64, tile * 128);
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
          asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
          mbar_arrive(&B.a_free[xb]);
        }
      }
    }
    if (leader) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    __syncwarp();
    tmem_dealloc_n(tmem, a.tmem_cols);
  }
}

// =================================================================== host
long long* g_ffn_trace = nullptr;
void ffn_set_trace(void* p) { g_ffn_trace = reinterpret_cast<long long*>(p); }
namespace {
bool ffn_fused_plan(int M, int C, int hid, ff::Args& a) {
  memset(&a, 0, sizeof(a));
  if (C % 16 || C > 384 || C < 16) return false;
  a.HC = C <= 256 ? 128 : 64;
  if (hid % a.HC) return false;
  if (C > 256 && (C / 2) % 16) return false;
  a.M = M;
  a.C = C;
  a.hid = hid;
  a.nch = hid / a.HC;
  a.tiles = (M + 127) / 128;
  a.slabs = (C + 63) / 64;
  a.u_bytes = a.slabs * a.HC * 128;
  a.v_bytes = (a.HC / 64) * C * 128;
  a.stage_bytes = std::max(a.u_bytes, a.v_bytes);
  a.us_bytes = a.HC * 128;
  a.vs_bytes = C * 128;
  const int avail = ff::kSmemMax - (int)sizeof(ff::Bars) - 64 - (hid + C) * 4;
  const int nus = a.nch * a.slabs, nvs = a.nch * (a.HC / 64);
  a.NA = 1;
  if (nus <= 16 && nvs <= 16 && a.slabs * 16384 + nus * a.us_bytes + nvs * a.vs_bytes <= avail) {
    a.resident = 1;  // every U / V slab stays in shared memory (C = 96: 168 KB)
    a.NU = nus;
    a.NV = nvs;
  } else {
    // streamed: x double-buffered when the rings still hold two chunks of each
    const int need = 2 * a.slabs * a.us_bytes + 2 * (a.HC / 64) * a.vs_bytes;
    a.NA = avail - 2 * a.slabs * 16384 >= need ? 2 : 1;
    int room = avail - a.NA * a.slabs * 16384;
    // two chunks of V slabs when they fit beside one chunk of U slabs (a
    // bulk copy takes ~2k cycles whatever its size, tools/probe_bulk_same.cu:
    // the ring depth sets the weight stream rate)
    a.NV = 2 * (a.HC / 64);
    while (a.NV > 1 && a.NV * a.vs_bytes + a.slabs * a.us_bytes > room) --a.NV;
    room -= a.NV * a.vs_bytes;
    a.NU = std::min(16, room / a.us_bytes);
    if (a.NU < 2 || a.NV < 1) return false;
  }
  a.direct = a.NA == 1;
  a.s_ring = a.NA * a.slabs * 16384;
  a.s_vring = a.s_ring + a.NU * a.us_bytes;
  a.stages = 0;
  a.stage_bytes = 0;
  a.t_z = 0;
  a.t_e = C;
  a.NE = C + 3 * a.HC <= 512 ? 3 : 2;
  const int cols = C + a.NE * a.HC;
  a.tmem_cols = 32;
  while (a.tmem_cols < (uint32_t)cols) a.tmem_cols *= 2;
  return a.tmem_cols <= 512;
}
using FfnK = void (*)(const CUtensorMap, const CUtensorMap, const CUtensorMap, const CUtensorMap, const CUtensorMap,
                      const ff::Args);
template <typename T>
FfnK ffn_kernel_t(int act) {
  switch (act) {
    case kRelu: return ffn_fused_kernel<kRelu, T>;
    case kSilu: return ffn_fused_kernel<kSilu, T>;
    case kSigmoid: return ffn_fused_kernel<kSigmoid, T>;
    case kGelu: return ffn_fused_kernel<kGelu, T>;
  }
  return ffn_fused_kernel<kIdentity, T>;
}
FfnK ffn_kernel_for(int act, int dtype) {
  return dtype == WL_DTYPE_BF16 ? ffn_kernel_t<__nv_bfloat16>(act) : ffn_kernel_t<__half>(act);
}
}  // namespace

bool ffn_fused_ok(int64_t M, int C, int hid) {
  ff::Args a;
  return M < (1ll << 31) && ffn_fused_plan((int)M, C, hid, a);
}

// x, res, z: [M][C] fp16; ut: [hid][C] fp16; vt: [C][hid] fp16; a: [hid], b: [C] fp32
int ffn_fused_run(const void* x, int64_t M, int C, int hid, const void* wimg, const float* abias, const float* bbias,
                  int act, const void* res, void* z, cudaStream_t st, int dtype) {
  ff::Args a;
  if (!ffn_fused_plan((int)M, C, hid, a)) return set_error(WL_EUNSUPPORTED, "fused FFN: no plan for C=%d hid=%d", C, hid);
  a.act = act;
  a.has_res = res != nullptr;
  a.a = abias;
  a.b = bbias;
  a.wimg = reinterpret_cast<const uint8_t*>(wimg);
  a.res = reinterpret_cast<const __half*>(res);
  a.z = reinterpret_cast<__half*>(z);
  a.trace = g_ffn_trace;
  auto map2 = [](CUtensorMap* m, const void* base, int inner, int64_t outer, int ld, int box_outer) {
    const uint64_t dims[2] = {(uint64_t)inner, (uint64_t)outer};
    const uint64_t strides[1] = {(uint64_t)ld * 2};
    const uint32_t box[2] = {64, (uint32_t)box_outer};
    return encode_tmap(m, base, 2, dims, strides, box, true);
  };
  CUtensorMap tx, tu, tv, tr, tz;
  if (int e = map2(&tx, x, C, M, C, 128)) return e;
  tu = tx;  // (weights arrive as bulk-copied images; the two map slots are unused)
  tv = tx;
  if (int e = map2(&tr, res ? res : x, C, M, C, 128)) return e;
  if (int e = map2(&tz, z, C, M, C, 128)) return e;
  const int smem = a.s_vring + a.NV * a.vs_bytes + ((int)sizeof(ff::Bars) + 15) / 16 * 16 + (hid + C) * 4;
  const int grid = a.tiles < kNumSMs ? a.tiles : kNumSMs;
  return launch_pdl(ffn_kernel_for(act, dtype), grid, ff::kThreads, smem, st, "ffn_fused launch", tx, tu, tv, tr, tz, a);
}

int64_t ffn_images_bytes(int C, int hid) {
  ff::Args a;
  if (!ffn_fused_plan(128, C, hid, a)) return 0;
  return (int64_t)a.nch * (a.u_bytes + a.v_bytes);
}

// u: reference (C, hid); v: reference (hid, C). Chunk j image: U_j as
// ceil(C/64) K-slabs of [HC rows][128 B], V_j as HC/64 K-slabs of [C rows][128 B],
// 16-byte chunk c of row n at n * 128 + ((c ^ n % 8) << 4) (the 128-byte swizzle)
void ffn_pack_images(int C, int hid, const float* u, const float* v, uint8_t* out, int dtype) {
  ff::Args a;
  if (!ffn_fused_plan(128, C, hid, a)) return;
  const int HC = a.HC;
  for (int j = 0; j < a.nch; ++j) {
    uint8_t* ui = out + (size_t)j * (a.u_bytes + a.v_bytes);
    uint8_t* vi = ui + a.u_bytes;
    for (int sl = 0; sl < a.slabs; ++sl)
      for (int n = 0; n < HC; ++n)
        for (int kk = 0; kk < 64; ++kk) {
          const int k = sl * 64 + kk;
          const float val = k < C ? u[(size_t)k * hid + j * HC + n] : 0.f;
          put_v(ui, (size_t)sl * HC * 128 + n * 128 + (((kk >> 3) ^ (n & 7)) << 4) + (kk & 7) * 2, val, dtype);
        }
    for (int sl = 0; sl < HC / 64; ++sl)
      for (int n = 0; n < C; ++n)
        for (int kk = 0; kk < 64; ++kk) {
          const int k = j * HC + sl * 64 + kk;
          put_v(vi, (size_t)sl * C * 128 + n * 128 + (((kk >> 3) ^ (n & 7)) << 4) + (kk & 7) * 2, v[(size_t)k * C + n],
                dtype);
        }
  }
}

int ffn_fused_init() {
  for (int dt : {WL_DTYPE_F16, WL_DTYPE_BF16})
    for (int act : {kIdentity, kRelu, kSilu, kSigmoid, kGelu})
      if (int e = check_cuda(cudaFuncSetAttribute(ffn_kernel_for(act, dt),
                                                  cudaFuncAttributeMaxDynamicSharedMemorySize, ff::kSmemMax),
                             "cudaFuncSetAttribute(ffn_fused)"))
        return e;
  return WL_OK;
}

}  // namespace wl
