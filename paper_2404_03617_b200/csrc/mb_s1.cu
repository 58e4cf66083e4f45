// mb_s1.cu — stride-1 MBConv + squeeze-excite with the grouped conv on the
// warp-level tensor path (core.py:112-122; fused schedule machine.py:649-733,
// layer-wise numerics machine.py:593-646). One CTA per image, one launch.
//
// Why two tensor paths: a tcgen05.mma costs max(~44, N/2) cycles per K=16
// step (profiles/r01_probe_mma_align.txt), so the T=8 grouped conv — N = 8
// output channels per group — can only reach it block-diagonally at 1/11 of
// the dense rate. The paper's own shape, mma.sync m16n8k{8,16} (K = 8 = T, no
// waste), runs on sm_100a at 1015 MAC/cycle/SM for k16 and overlaps with
// tcgen05 issued by another warp (profiles/r02_probe_hmma.txt). So:
//   tcgen05 (one issuing thread)   : expand  E_j = x . W_exp[:, j]   (SS, TMEM)
//                                    project Z  += h2_j' . W_prj[j]  (SS, TMEM)
//   mma.sync (8 conv warps)        : h2_j = phi(conv3x3_T8(h1_j) + b_conv)
//                                    from ldmatrix fragments of h1 in smem
// Geometry: the image sits in a flat padded layout of row pitch 16 (W <= 14):
// flat row m = 16 y + i holds pixel (y, i - 1); i = 0 and i > W are zero pads.
// An m16 HMMA fragment is one padded image row, so the three input rows of a
// 3x3 tap window slide down the image and every ldmatrix fragment is used by
// three output rows. x arrives by one TMA box per 64 channels ({64, 16, H}
// from x = -1: OOB columns zero-filled, 128B-swizzled = the tcgen05 A layout);
// z leaves through the same map from x = 0 (the OOB pad columns are dropped).
//
// Phases per CTA (hidden chunks of 64 = 8 groups):
//   A  producer: x, biases, W_exp ring     MMA: expand chunk j -> E[j%2]
//      E warps (8): E + b_exp, phi -> h1[j%2] (padded image, per-group planes)
//      conv warps (8, one group each): HMMA conv + b_conv, phi -> registers,
//      SE pool in registers; h2_j stored (whole 128-byte lines per warp store)
//      to the L2-resident workspace in the projection's A layout (the tensor
//      machine's GLOBAL tier, machine.py:667-687)
//   B  conv warps: squeeze-excite gates (pool -> W_sq, ReLU -> W_ex, sigmoid)
//   C  producer reloads h2 + W_prj by half-chunks (4-slot ring over the dead
//      h1 / W_exp buffers); conv warps gate them in place; MMA: Z += h2' . W_prj
//   D  E warps: z = Z + b_prj + x (in place over the x tile) -> TMA store
// Stage mode (nblk > 1, the paper's per-stage persistence, machine.py:1091-1120 /
// PAPER.md:1328-1347): the CTA runs nblk consecutive stride-1 blocks of its
// image; block b's z stays in the x tile in shared memory as block b+1's input
// (only the stage's first input and last output cross HBM), the next block's
// header and W_ex land after phase D, and every barrier keeps counting phases
// across blocks.
#include <cuda.h>
#include <cuda_fp16.h>
#include <cstdint>
#include <cstring>
#include "common.cuh"
#include "plan.h"

namespace wl {

constexpr int kMb1MaxStage = 20;
struct Mb1Args {
  int n, H, W, C, hid, sq, nch, NT;
  int K;  // output channels (C for stride 1; stride 2: 64 or 128)
  int s_x, s_h1, s_h1_bytes, s_w, s_wex, s_hdr, s_se, s_bar, smem;
  int hdr_stride;
  int s_h2;  // P = 8: the block's whole h2 (compact 64-row chunks) stays in shared memory
  int o_bexp, o_bconv, o_bprj, hdr_bytes;  // header (fp32) in the packed blob
  int64_t o_se, o_frag, o_wexp, o_wprj;    // packed-blob sections
  int o_bsq, o_wex, o_bex;                 // inside the SE section (fp16 matrices, fp32 biases)
  int t_e, t_z, tmem_cols;
  int slot_bytes;  // phase C ring slot: h2 half-chunk (NT x 8 KB) + W_prj half-chunk (C x 32 x 2)
  const uint8_t* wpack;
  int nblk;                           // consecutive blocks run by this launch (a stage)
  const uint8_t* wpacks[kMb1MaxStage];  // their packed blobs (nblk > 1)
  uint8_t* h2;  // workspace: [n][nch][NT][8 groups][128 rows][16 B]
  long long* trace;
};

namespace mb1 {
constexpr int kWarps = 18;
constexpr int kThreads = kWarps * 32;
constexpr int kProd = 0, kMma = 1, kE0 = 2, kC0 = 10;
constexpr int kHC = 64;  // hidden channels per chunk (8 groups of T = 8)
struct Bars {
  uint64_t x_full, hdr_full[2];  // hdr double-buffered: block b + 1's header lands during block b
  uint64_t w_full[2], w_empty[2];
  uint64_t e_full[2], e_empty[2];
  uint64_t h1_full[2], h1_empty[2];
  uint64_t a_done;
  uint64_t pa_full[4], pa_ready[4], pa_empty[4];
  uint64_t z_full, se_full;
  uint64_t sq_full;      // the E warps' squeeze outputs are in shared memory
  uint64_t pool_full[2];  // a chunk's pooled sums are in shared memory
  uint64_t d_done;  // stage: block b's output tile is in place (x of block b + 1), hdr / W_ex free
  uint32_t tmem_base;
};
}  // namespace mb1

__device__ __forceinline__ void tma_load_4d(void* dst, const void* tmap, int c0, int c1, int c2, int c3,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, "
      "%5}], [%6];" ::"r"(smem_u32(dst)),
      "l"(tmap), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_store_4d(const void* tmap, const void* src, int c0, int c1, int c2, int c3) {
  asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%2, %3, %4, %5}], [%1];" ::"l"(tmap),
               "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
               : "memory");
}
__device__ __forceinline__ void bulk_commit_s1() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0_s1() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait0_s1() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)),
               "r"(bytes)
               : "memory");
}

#define MB1_TRACE(slot)                                                  \
  do {                                                                   \
    if (a.trace && blockIdx.x == 0) a.trace[(slot)] = clock64();         \
  } while (0)

// flat-layout row pitch: 16 (W <= 15) or, for the 7x7 stage, 8 — row y's
// right pad is row y + 1's left pad, so one m16 fragment covers two image rows
// and the conv needs 4 fragments instead of 7
__host__ __device__ constexpr int mb1_pitch(int h) { return h <= 7 ? 8 : 16; }
// bytes of one h1 group plane: the flat image (16-row fragments), one zero image
// row above, the rows the last fragment's dy = +1 / dx = +1 loads reach, margins
__host__ __device__ constexpr int mb1_plane_bytes(int h) {
  return (16 * ((mb1_pitch(h) * h + 15) / 16) + 3 * mb1_pitch(h) + 2) * 16;
}

// H: image rows (flat rows P H <= 128 NT); C: block channels (64 or 128)
// S2: the stride-2 block (H = 14 -> 7): the conv output is blurred (Triangle-3,
// stride 2, reflect) in the conv warps' registers and h2 is stored at 7 x 7 in
// the compact pitch-8 layout; SE, projection (M = 64) and the output run at
// 7 x 7, without a shortcut (PAPER.md BlurPool downsampling; complexity.py:208-215)
template <int H, int C, int ACT, bool S2>
__global__ void __launch_bounds__(mb1::kThreads, 1)
    mb_s1_kernel(const __grid_constant__ CUtensorMap tmap_x, const __grid_constant__ CUtensorMap tmap_z,
                 const __grid_constant__ Mb1Args a) {
  using namespace mb1;
  constexpr int P = mb1_pitch(H);            // flat row pitch
  constexpr int NT = (P * H + 127) / 128;    // M tiles of the flat image
  constexpr int KH = C / 64;                 // 64-channel (128-byte) halves of x
  constexpr int XH = NT * 128 * 128;         // bytes of one x half
  constexpr int GS = mb1_plane_bytes(H);     // bytes of one h1 group plane
  static_assert(P * H <= 256 && (C == 64 || C == 128), "geometry");
  // P = 8: the 16-row fragments of the flat image sit at A rows 32 k .. 32 k + 15
  // (one per TMEM lane quadrant), so the expand and projection accumulators
  // spread over all four quadrants and every epilogue warp has rows to drain
  // (a flat 56-row image would leave quadrants 2 and 3 — and their warps — idle)
  auto flat_of = [](int arow) -> int {
    if constexpr (P == 8) return (arow & 31) < 16 ? (arow >> 5) * 16 + (arow & 15) : (1 << 20);
    return arow;
  };
  static_assert(P == 16 || P * H <= 64, "P = 8 holds at most four 16-row fragments");
  static_assert(!S2 || (H == 14 && P == 16), "stride-2 variant: 14x14 -> 7x7");
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* s_x = smem + a.s_x;
  uint8_t* s_h1 = smem + a.s_h1;   // 2 buffers x 8 group planes; phase C ring overlays s_h1 .. s_w end
  uint8_t* s_w = smem + a.s_w;     // W_exp ring, 2 x (64 x C fp16)
  uint8_t* s_hdr0 = smem + a.s_hdr;  // two header buffers of a.hdr_stride bytes
  auto hdr_of = [&](int blk) -> uint8_t* { return s_hdr0 + (blk & 1) * a.hdr_stride; };
  uint8_t* s_se = smem + a.s_se;   // pool f32[hid] | gates h2[hid/2] | scratch f32[256 + 32]
  uint8_t* s_wex = smem + a.s_wex; // W_ex (sq x hid fp16), prefetched for the excite
  Bars& B = *reinterpret_cast<Bars*>(smem + a.s_bar);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int img = blockIdx.x;
  const int nch = a.nch;
  const int nblk = a.nblk;
  auto wp_of = [&](int blk) -> const uint8_t* { return nblk > 1 ? a.wpacks[blk] : a.wpack; };

  if (threadIdx.x == 0) {
    mbar_init(&B.x_full, 1);
    mbar_init(&B.hdr_full[0], 1);
    mbar_init(&B.hdr_full[1], 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&B.w_full[i], 1);
      mbar_init(&B.w_empty[i], 1);
      mbar_init(&B.e_full[i], 1);
      mbar_init(&B.e_empty[i], 256);
      mbar_init(&B.h1_full[i], 256);
      mbar_init(&B.h1_empty[i], 256);
    }
    for (int i = 0; i < 4; ++i) {
      mbar_init(&B.pa_full[i], 1);
      mbar_init(&B.pa_ready[i], 256);
      mbar_init(&B.pa_empty[i], 1);
    }
    mbar_init(&B.a_done, 1);
    mbar_init(&B.z_full, 1);
    mbar_init(&B.se_full, 1);
    mbar_init(&B.sq_full, 32);
    mbar_init(&B.pool_full[0], 256);
    mbar_init(&B.pool_full[1], 256);
    mbar_init(&B.d_done, 256);
    fence_mbar_init();
  }
  if (warp == kMma) tmem_alloc_n(&B.tmem_base, a.tmem_cols);
  // zero the h1 planes (halo rows / margins stay zero for phase A) and the pool
  for (int i = threadIdx.x; i < (2 * 8 * GS) / 16; i += kThreads)
    reinterpret_cast<uint4*>(s_h1)[i] = make_uint4(0, 0, 0, 0);
  for (int i = threadIdx.x; i < a.hid; i += kThreads) reinterpret_cast<float*>(s_se)[i] = 0.f;
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  pdl_trigger();
  pdl_wait();
  const uint32_t tmem = B.tmem_base;
  MB1_TRACE(0);

  if (warp == kProd) {
    if (lane == 0) {
      // ------------------------------------------------------------ producer
      prefetch_tmap(&tmap_x);
      const uint32_t wbytes = kHC * C * 2, vbytes = C * 32 * 2;
      const uint8_t* h2img = a.h2 + (size_t)img * nch * NT * 16384;
      auto load_hdr = [&](int b) {
        mbar_arrive_expect_tx(&B.hdr_full[b & 1], a.hdr_bytes);
        bulk_g2s(hdr_of(b), wp_of(b), a.hdr_bytes, &B.hdr_full[b & 1]);
      };
      auto load_wexp = [&](int b, int j) {
        const int g = b * nch + j, wb = g & 1, u = g >> 1;
        mbar_wait(&B.w_empty[wb], (u & 1) ^ 1);
        mbar_arrive_expect_tx(&B.w_full[wb], wbytes);
        bulk_g2s(s_w + wb * wbytes, wp_of(b) + a.o_wexp + (size_t)j * wbytes, wbytes, &B.w_full[wb]);
      };
      int pre = 0;  // W_exp chunks of this block already issued during the previous one
      load_hdr(0);
      for (int blk = 0; blk < nblk; ++blk) {
        const uint8_t* wp = wp_of(blk);
        if (blk > 0) mbar_wait(&B.d_done, (blk - 1) & 1);  // previous block's phase D done: W_ex, x free
        // the other header buffer was block blk - 1's: free after its phase D
        if (blk + 1 < nblk) load_hdr(blk + 1);
        if (blk == 0) {
          mbar_arrive_expect_tx(&B.x_full, P == 8 ? KH * ((H + 1) / 2) * 2048 : KH * 64 * 2 * P * H);
          if constexpr (P == 8) {
            for (int kh = 0; kh < KH; ++kh)
              for (int k = 0; k < (H + 1) / 2; ++k)
                tma_load_4d(s_x + kh * XH + k * 2048, &tmap_x, kh * 64, -1, 2 * k, img, &B.x_full);
          } else {
            for (int kh = 0; kh < KH; ++kh) tma_load_4d(s_x + kh * XH, &tmap_x, kh * 64, -1, 0, img, &B.x_full);
          }
        } else {
          mbar_arrive(&B.x_full);  // the previous block's z, in place (its writers fenced before d_done)
        }
        mbar_arrive_expect_tx(&B.se_full, a.sq * a.hid * 2);
        bulk_g2s(s_wex, wp + a.o_se + a.o_wex, a.sq * a.hid * 2, &B.se_full);
        for (int j = pre; j < nch; ++j) load_wexp(blk, j);
        pre = 0;
        // phase C: h2 chunks come back once phase A stored them all and released
        // the h1 / W_exp buffers the ring overlays
        // ring of 4 half-chunks (32 hidden channels: NT x 8 KB of h2 + the
        // matching 4 K-columns of W_prj), so several reloads are in flight
        if constexpr (P == 8) {
          // h2 stays in shared memory: the ring streams W_prj chunks only (K = 64).
          // Chunks 0 / 1 go to the W_exp buffers (free once the last two expands
          // completed, before the conv ends), chunks 2 / 3 to the h1 buffers
          for (int j = 0; j < nch; ++j) {
            const int gq = blk * nch + j;
            const int s = gq & 3, u = gq >> 2;
            mbar_wait(&B.pa_empty[s], (u & 1) ^ 1);
            if (j < 2) {
              const int gl = blk * nch + nch - 2 + j;  // last expand that used W buffer j
              mbar_wait(&B.w_empty[gl & 1], (gl >> 1) & 1);
            } else if (j < 4) {
              mbar_wait(&B.a_done, blk & 1);
            }
            mbar_arrive_expect_tx(&B.pa_full[s], 2 * vbytes);
            bulk_g2s(s_w + s * a.slot_bytes, wp + a.o_wprj + (size_t)j * 2 * vbytes, 2 * vbytes,
                     &B.pa_full[s]);
          }
        } else if constexpr (S2) {
          // 7x7 h2 chunks (compact, 8 KB) + W_prj chunks (K x 64) through the ring
          const uint32_t zbytes = a.K * kHC * 2;
          mbar_wait(&B.a_done, blk & 1);
          for (int j = 0; j < nch; ++j) {
            const int gq = blk * nch + j;
            const int s = gq & 3, u = gq >> 2;
            mbar_wait(&B.pa_empty[s], (u & 1) ^ 1);
            uint8_t* slot = s_h1 + s * a.slot_bytes;
            mbar_arrive_expect_tx(&B.pa_full[s], 8192 + zbytes);
            bulk_g2s(slot, a.h2 + ((size_t)img * nch + j) * 8192, 8192, &B.pa_full[s]);
            bulk_g2s(slot + 8192, wp + a.o_wprj + (size_t)j * zbytes, zbytes, &B.pa_full[s]);
          }
        } else {
        mbar_wait(&B.a_done, blk & 1);
        for (int qq = 0; qq < 2 * nch; ++qq) {
          const int gq = blk * 2 * nch + qq;
          const int s = gq & 3, u = gq >> 2, j = qq >> 1, half = qq & 1;
          mbar_wait(&B.pa_empty[s], (u & 1) ^ 1);
          uint8_t* slot = s_h1 + s * a.slot_bytes;
          mbar_arrive_expect_tx(&B.pa_full[s], NT * 8192 + vbytes);
          for (int t = 0; t < NT; ++t)
            bulk_g2s(slot + t * 8192, h2img + ((size_t)j * NT + t) * 16384 + half * 8192, 8192, &B.pa_full[s]);
          bulk_g2s(slot + NT * 8192, wp + a.o_wprj + (size_t)j * 2 * vbytes + half * vbytes, vbytes,
                   &B.pa_full[s]);
        }
        }
        if (blk + 1 < nblk) {
          // the next block's first W_exp chunks go into the W ring as soon as the
          // phase C ring overlaying it is consumed (its last projection MMAs
          // committed), not after phase D: the next expand starts at d_done
          const int gl = P == 8 ? blk * nch + nch - 1 : blk * 2 * nch + 2 * nch - 1;
          mbar_wait(&B.pa_empty[gl & 3], (gl >> 2) & 1);
          pre = nch < 2 ? nch : 2;
          for (int j = 0; j < pre; ++j) load_wexp(blk + 1, j);
        }
      }
    }
  } else if (warp == kMma) {
    {  // the whole warp runs the issue loop; one elected lane issues each MMA / commit
      // ------------------------------------------------------------ MMA issuer
      // P = 8: M = 64 over the compact 64-row x tile; the accumulator rows land
      // 16 per TMEM lane quadrant (rows 16k.. at lanes 32k..)
      const uint32_t idesc_e = make_idesc_f16(P == 8 ? 64 : 128, kHC);
      const uint32_t idesc_z = make_idesc_f16(128, C);
      const uint32_t wbytes = kHC * C * 2;
      for (int blk = 0; blk < nblk; ++blk) {
        mbar_wait(&B.x_full, blk & 1);
        tc_fence_after();
        if (lane == 0) MB1_TRACE(70);
        for (int j = 0; j < nch; ++j) {
          const int g = blk * nch + j, b = g & 1, u = g >> 1;
          mbar_wait(&B.w_full[b], u & 1);
          mbar_wait(&B.e_empty[b], (u & 1) ^ 1);
          tc_fence_after();
          if (lane == 0) MB1_TRACE(36 + j);
          const uint32_t wb = smem_u32(s_w + b * wbytes);
#pragma unroll
          for (int t = 0; t < NT; ++t)
#pragma unroll
            for (int k = 0; k < C / 16; ++k) {
              const uint64_t ad = make_sdesc_sw128(smem_u32(s_x) + (k / 4) * XH + t * 16384 + (k % 4) * 32);
              const uint64_t bd = make_sdesc(wb + k * 2 * 1024, 1024, 128);
              mma_ss_w(tmem + a.t_e + (b * NT + t) * kHC, ad, bd, idesc_e, k > 0);
            }
          mma_commit_w(&B.e_full[b]);
          mma_commit_w(&B.w_empty[b]);
        }
        // Z of the previous block must have been drained (phase D) before the
        // first projection of this one overwrites it: d_done(blk - 1) precedes
        // x_full(blk), waited above
        if constexpr (P == 8) {
          const uint32_t idesc_z64 = make_idesc_f16(64, C);
          for (int j = 0; j < nch; ++j) {
            const int gq = blk * nch + j;
            const int s = gq & 3, u = gq >> 2;
            mbar_wait(&B.pa_full[s], u & 1);   // W_prj chunk landed
            mbar_wait(&B.pa_ready[s], u & 1);  // h2 chunk gated
            tc_fence_after();
            if (lane == 0) MB1_TRACE(52 + j);
            const uint32_t vb = smem_u32(s_w + s * a.slot_bytes);
            const uint32_t hb = smem_u32(smem + a.s_h2) + j * 8192;
#pragma unroll
            for (int k = 0; k < kHC / 16; ++k) {
              const uint64_t ad = make_sdesc(hb + k * 2 * 1024, 1024, 128);
              const uint64_t bd = make_sdesc(vb + k * 2 * (C / 8) * 128, (C / 8) * 128, 128);
              mma_ss_w(tmem + a.t_z, ad, bd, idesc_z64, (j > 0 || k > 0));
            }
            mma_commit_w(&B.pa_empty[s]);
          }
        } else if constexpr (S2) {
          const uint32_t idesc_s2 = make_idesc_f16(64, a.K);
          for (int j = 0; j < nch; ++j) {
            const int gq = blk * nch + j;
            const int s = gq & 3, u = gq >> 2;
            mbar_wait(&B.pa_ready[s], u & 1);  // landed and gated
            tc_fence_after();
            if (lane == 0) MB1_TRACE(52 + j);
            const uint32_t slot = smem_u32(s_h1 + s * a.slot_bytes);
#pragma unroll
            for (int k = 0; k < kHC / 16; ++k) {
              const uint64_t ad = make_sdesc(slot + k * 2 * 1024, 1024, 128);
              const uint64_t bd = make_sdesc(slot + 8192 + k * 2 * (a.K / 8) * 128, (a.K / 8) * 128, 128);
              mma_ss_w(tmem + a.t_z, ad, bd, idesc_s2, (j > 0 || k > 0));
            }
            mma_commit_w(&B.pa_empty[s]);
          }
        } else {
        for (int qq = 0; qq < 2 * nch; ++qq) {
          const int gq = blk * 2 * nch + qq;
          const int s = gq & 3, u = gq >> 2;
          mbar_wait(&B.pa_ready[s], u & 1);
          tc_fence_after();
          if (!(qq & 1)) if (lane == 0) MB1_TRACE(52 + (qq >> 1));
          const uint32_t slot = smem_u32(s_h1 + s * a.slot_bytes);
          const uint32_t vb = slot + NT * 8192;
#pragma unroll
          for (int t = 0; t < NT; ++t)
#pragma unroll
            for (int k = 0; k < 2; ++k) {
              const uint64_t ad = make_sdesc(slot + t * 8192 + k * 2 * 2048, 2048, 128);
              const uint64_t bd = make_sdesc(vb + k * 2 * (C / 8) * 128, (C / 8) * 128, 128);
              mma_ss_w(tmem + a.t_z + t * C, ad, bd, idesc_z, (qq > 0 || k > 0));
            }
          mma_commit_w(&B.pa_empty[s]);
        }
        }
        mma_commit_w(&B.z_full);
      }
    }
  } else if (warp < kC0) {
    // ---------------------------------------------- E warps: expand epilogue
    const int e = warp - kE0, q = warp & 3, hh = e >> 2;  // TMEM lane quadrant = warp % 4
    const float* s_bexp = nullptr;
    const float* s_bprj = nullptr;
    for (int blk = 0; blk < nblk; ++blk) {
      // squeeze partials, chunk by chunk as the conv warps pool them (the E
      // warps idle while the conv runs): thread (warp e, lane o) accumulates
      // W_sq[c][o] pool[c] over its 8 channels c of every chunk, fixed order;
      // its W_sq^T row segment is loaded one chunk ahead
      const __half* wsqt = reinterpret_cast<const __half*>(wp_of(blk) + a.o_se);
      const float* pool = reinterpret_cast<const float*>(s_se);
      float sq_acc = 0.f;
      // W_sq^T segments of chunks jj (in wq) and jj + 1 (wq_next): each load is
      // issued a whole chunk before its use
      uint4 wq = ldg_pinned(wsqt + (size_t)lane * a.hid + e * 8);
      uint4 wq_next = nch > 1 ? ldg_pinned(wsqt + (size_t)lane * a.hid + kHC + e * 8) : wq;
      auto squeeze_part = [&](int jj) {
        const int gg = blk * nch + jj;
        mbar_wait(&B.pool_full[gg & 1], (gg >> 1) & 1);
        const float4 pa = *reinterpret_cast<const float4*>(pool + jj * kHC + e * 8);
        const float4 pb = *reinterpret_cast<const float4*>(pool + jj * kHC + e * 8 + 4);
        const __half* w8 = reinterpret_cast<const __half*>(&wq);
        sq_acc = fmaf(pa.x, __half2float(w8[0]), sq_acc);
        sq_acc = fmaf(pa.y, __half2float(w8[1]), sq_acc);
        sq_acc = fmaf(pa.z, __half2float(w8[2]), sq_acc);
        sq_acc = fmaf(pa.w, __half2float(w8[3]), sq_acc);
        sq_acc = fmaf(pb.x, __half2float(w8[4]), sq_acc);
        sq_acc = fmaf(pb.y, __half2float(w8[5]), sq_acc);
        sq_acc = fmaf(pb.z, __half2float(w8[6]), sq_acc);
        sq_acc = fmaf(pb.w, __half2float(w8[7]), sq_acc);
        wq = wq_next;
        if (jj + 2 < nch) wq_next = ldg_pinned(wsqt + (size_t)lane * a.hid + (jj + 2) * kHC + e * 8);
      };
      mbar_wait(&B.hdr_full[blk & 1], (blk >> 1) & 1);
      s_bexp = reinterpret_cast<const float*>(hdr_of(blk) + a.o_bexp);
      s_bprj = reinterpret_cast<const float*>(hdr_of(blk) + a.o_bprj);
      for (int j = 0; j < nch; ++j) {
        const int g2 = blk * nch + j, b = g2 & 1, u = g2 >> 1;
        mbar_wait(&B.e_full[b], u & 1);
        mbar_wait(&B.h1_empty[b], (u & 1) ^ 1);
        tc_fence_after();
        uint8_t* h1 = s_h1 + b * 8 * GS;
        if constexpr (P == 8) {
          // the quadrant's 16 real A rows spread over all 32 threads (16x256b):
          // every lane converts 16 values instead of half the lanes converting 32
          uint32_t v[16];
          WL_TMEM_LD_16x256b_X4(tmem_lane_addr(tmem, q, a.t_e + b * NT * kHC + hh * 32), v);
          tmem_ld_wait();
          const int r0 = lane >> 2, c2 = (lane & 3) * 2;
          const int f0 = 16 * q + r0, f1 = f0 + 8;  // flat rows
          const bool ok0 = f0 < P * H && (f0 & 7) >= 1 && (f0 & 7) <= a.W;
          const bool ok1 = f1 < P * H && (f1 & 7) >= 1 && (f1 & 7) <= a.W;
          const float* bb = s_bexp + j * kHC + hh * 32 + c2;
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const float2 bv = *reinterpret_cast<const float2*>(bb + 8 * k);
            __half2 h0 = act_h2<ACT>(__floats2half2_rn(__uint_as_float(v[4 * k]) + bv.x,
                                                       __uint_as_float(v[4 * k + 1]) + bv.y));
            __half2 h1v = act_h2<ACT>(__floats2half2_rn(__uint_as_float(v[4 * k + 2]) + bv.x,
                                                        __uint_as_float(v[4 * k + 3]) + bv.y));
            if (!ok0) h0 = __float2half2_rn(0.f);
            if (!ok1) h1v = __float2half2_rn(0.f);
            uint8_t* pl = h1 + (hh * 4 + k) * GS + c2 * 2;
            if (f0 < P * H) *reinterpret_cast<__half2*>(pl + (f0 + P + 1) * 16) = h0;
            if (f1 < P * H) *reinterpret_cast<__half2*>(pl + (f1 + P + 1) * 16) = h1v;
          }
        } else {
#pragma unroll
        for (int t = 0; t < NT; ++t) {
          uint32_t v[32];
          const uint32_t ta = tmem_lane_addr(tmem, q, a.t_e + (b * NT + t) * kHC + hh * 32);
          WL_TMEM_LD16(ta, v);
          WL_TMEM_LD16(ta + 16, (v + 16));
          tmem_ld_wait();
          const int m = flat_of(t * 128 + q * 32 + lane);
          const int i = m & (P - 1);
          if (m < P * H) {
            const bool real = i >= 1 && i <= a.W;
            const float* bb = s_bexp + j * kHC + hh * 32;
#pragma unroll
            for (int g = 0; g < 4; ++g) {
              const uint4 val = real ? bias_act8<ACT>(v + 8 * g, bb + 8 * g) : make_uint4(0, 0, 0, 0);
              *reinterpret_cast<uint4*>(h1 + (hh * 4 + g) * GS + (m + P + 1) * 16) = val;
            }
          }
        }
        }
        tc_fence_before();
        mbar_arrive(&B.e_empty[b]);
        mbar_arrive(&B.h1_full[b]);
        if (e == 0 && lane == 0) MB1_TRACE(4 + j);
        // chunk j - 2's pool was written after conv(j - 2) released h1[b], so
        // it is (nearly) complete here, and h1(j) is already out
        if (j >= 2) squeeze_part(j - 2);
      }
      // ---------------------------------------------- phase B (squeeze)
      for (int jj = nch >= 2 ? nch - 2 : 0; jj < nch; ++jj) squeeze_part(jj);
      {
        float* scr = reinterpret_cast<float*>(s_se + a.hid * 4 + a.hid * 2);
        const float bsq_o = lane < a.sq ? reinterpret_cast<const float*>(wp_of(blk) + a.o_se + a.o_bsq)[lane] : 0.f;
        scr[e * 32 + lane] = sq_acc;
        nbar(3, 256);
        if (e == 0) {
          float sv = 0.f;
#pragma unroll
          for (int r = 0; r < 8; ++r) sv += scr[r * 32 + lane];
          const float inv_p = S2 ? 1.f / (float)((a.H / 2) * (a.W / 2)) : 1.f / (float)(a.H * a.W);
          scr[256 + lane] = lane < a.sq ? fmaxf(sv * inv_p + bsq_o, 0.f) : 0.f;
          mbar_arrive(&B.sq_full);
        }
      }
      // ---------------------------------------------- phase D: z epilogue
      mbar_wait(&B.z_full, blk & 1);
      tc_fence_after();
      if (e == 0 && lane == 0) MB1_TRACE(68);
      if constexpr (S2) {
        // Z (M = 64): 7x7 compact row 16 q + lane at TMEM lane 32 q + lane; the
        // x tile is dead (no shortcut), so z is staged over it
        const int f = 16 * q + lane;
        if (hh < a.K / 64) {
          uint32_t v[64];
          const uint32_t za = tmem_lane_addr(tmem, q, a.t_z + hh * 64);
          WL_TMEM_LD16(za, v);
          WL_TMEM_LD16(za + 16, (v + 16));
          WL_TMEM_LD16(za + 32, (v + 32));
          WL_TMEM_LD16(za + 48, (v + 48));
          tmem_ld_wait();
          if (lane < 16 && f < 56) {
            uint8_t* zrow = s_x + hh * XH + f * 128;
#pragma unroll
            for (int c8 = 0; c8 < 8; ++c8) {
              const float4 b0 = *reinterpret_cast<const float4*>(s_bprj + hh * 64 + c8 * 8);
              const float4 b1 = *reinterpret_cast<const float4*>(s_bprj + hh * 64 + c8 * 8 + 4);
              const float bb[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
              float fz[8];
#pragma unroll
              for (int r = 0; r < 8; ++r) fz[r] = __uint_as_float(v[c8 * 8 + r]) + bb[r];
              *reinterpret_cast<uint4*>(zrow + ((c8 ^ (f & 7)) << 4)) = pack8(fz);
            }
          }
        }
      } else if (hh < KH) {
#pragma unroll 1
        for (int t = 0; t < NT; ++t) {
          const int m = t * 128 + q * 32 + lane;  // A row (TMEM lane)
          const int xr = P == 8 ? flat_of(m) & 63 : m;  // x / z tile row (P = 8: compact)
          uint8_t* xrow = s_x + hh * XH + xr * 128;
          uint32_t v[64];  // the row's 64 channels in one batch of TMEM loads
          const uint32_t za = tmem_lane_addr(tmem, q, a.t_z + t * C + hh * 64);
          WL_TMEM_LD16(za, v);
          WL_TMEM_LD16(za + 16, (v + 16));
          WL_TMEM_LD16(za + 32, (v + 32));
          WL_TMEM_LD16(za + 48, (v + 48));
          tmem_ld_wait();
          if (flat_of(m) < P * H) {
#pragma unroll
            for (int c8 = 0; c8 < 8; ++c8) {
              uint8_t* p = xrow + ((c8 ^ (xr & 7)) << 4);
              float res[8];
              unpack8(lds128(p), res);
              const float4 b0 = *reinterpret_cast<const float4*>(s_bprj + hh * 64 + c8 * 8);
              const float4 b1 = *reinterpret_cast<const float4*>(s_bprj + hh * 64 + c8 * 8 + 4);
              const float bb[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
              float f[8];
#pragma unroll
              for (int r = 0; r < 8; ++r) f[r] = __uint_as_float(v[c8 * 8 + r]) + bb[r] + res[r];
              *reinterpret_cast<uint4*>(p) = pack8(f);
            }
          }
        }
      }
      if (blk + 1 < nblk) {
        // the phase C ring overlaid the h1 planes: restore their zero halo
        // rows / margins for the next block's conv
        for (int i = threadIdx.x - kE0 * 32; i < (2 * 8 * GS) / 16; i += 256)
          reinterpret_cast<uint4*>(s_h1)[i] = make_uint4(0, 0, 0, 0);
      }
      tc_fence_before();
      fence_async_smem();
      mbar_arrive(&B.d_done);  // z (the next block's x) written and fenced; hdr / W_ex / ring free
      if (blk + 1 == nblk) {
        nbar(2, 256);
        if (e == 0 && lane == 0) {
          // a TMA store may not start at a negative coordinate (illegal instruction,
          // tools/probe_tma_store.cu): start at x = 0 one 128-byte row into the tile
          // (the 128B swizzle is address-based, so the shifted source stays valid)
          if constexpr (S2) {
            for (int kh = 0; kh < a.K / 64; ++kh)
              for (int k = 0; k < 4; ++k) tma_store_4d(&tmap_z, s_x + kh * XH + k * 2048 + 128, kh * 64, 0, 2 * k, img);
          } else if constexpr (P == 8) {
            for (int kh = 0; kh < KH; ++kh)
              for (int k = 0; k < (H + 1) / 2; ++k)
                tma_store_4d(&tmap_z, s_x + kh * XH + k * 2048 + 128, kh * 64, 0, 2 * k, img);
          } else {
            for (int kh = 0; kh < KH; ++kh) tma_store_4d(&tmap_z, s_x + kh * XH + 128, kh * 64, 0, 0, img);
          }
          bulk_commit_s1();
          bulk_wait_read0_s1();  // the tile must outlive the reads only; the writes complete on their own
          MB1_TRACE(69);
        }
      }
    }
  } else {
    // ------------------------------------------ conv warps: HMMA 3x3 T=8 conv
    const int g = warp - kC0;  // group within the chunk
    const int tid = threadIdx.x - kC0 * 32;
    const int gid = lane >> 2, tq = lane & 3;
    const int sq = a.sq, hid = a.hid;
    const float* s_bconv = nullptr;
    const uint32_t lrow = (lane & 15), lsel = lane >> 4;  // ldmatrix: row of the fragment, which fragment
    uint8_t* h2img = a.h2 + (size_t)img * nch * NT * 16384;
    const __half2 one2 = __float2half2_rn(1.f), zero2 = __float2half2_rn(0.f);
    // real pixels among the fragment rows gid / gid + 8 (the pads are zero)
    const __half2 m0 = (gid >= 1 && gid <= a.W) ? one2 : zero2,
                  m1 = P == 16 ? ((gid + 8 <= a.W) ? one2 : zero2) : m0;
    for (int blk = 0; blk < nblk; ++blk) {
    const uint8_t* wp = wp_of(blk);
    const uint32_t* frag = reinterpret_cast<const uint32_t*>(wp + a.o_frag);
    // B fragments in pair order (t0,t1) (t3,t4) (t6,t7) (t2,t5) t8: each k16
    // pair is two consecutive registers (mb1_pack)
    uint32_t bw[9];
#pragma unroll
    for (int tp = 0; tp < 9; ++tp) bw[tp] = __ldg(frag + ((size_t)(0 * 8 + g) * 9 + tp) * 32 + lane);
    mbar_wait(&B.hdr_full[blk & 1], (blk >> 1) & 1);
    s_bconv = reinterpret_cast<const float*>(hdr_of(blk) + a.o_bconv);
    // excite biases of this thread's first gate pair, needed after phase A
    const float2 bex_pre = tid < hid / 2 ? __ldg(reinterpret_cast<const float2*>(wp + a.o_se + a.o_bex) + tid)
                                         : make_float2(0.f, 0.f);
    for (int j = 0; j < nch; ++j) {
      const int g2 = blk * nch + j, b = g2 & 1, u = g2 >> 1;
      if (tid == 0) MB1_TRACE(72 + j);
      const float2 bc = *reinterpret_cast<const float2*>(s_bconv + j * kHC + g * 8 + tq * 2);
      // next chunk's B fragments: a whole chunk of conv work hides their L2 latency
      uint32_t bwn[9];
      if (j + 1 < nch) {
#pragma unroll
        for (int tp = 0; tp < 9; ++tp) bwn[tp] = __ldg(frag + ((size_t)((j + 1) * 8 + g) * 9 + tp) * 32 + lane);
      }
      if (tid == 0) MB1_TRACE(80 + j);
      mbar_wait(&B.h1_full[b], u & 1);
      if (tid == 0) MB1_TRACE(12 + j);
      const uint32_t plane = smem_u32(s_h1 + b * 8 * GS + g * GS) + 16;  // + 1 margin row
      // row unit r = P flat rows (one padded image row). Q_r: x4 at unit r,
      // dx = -1 (lanes 0-15) and dx = 0 (lanes 16-31); P_r: x4 of dx = +1 at
      // units r (lanes 0-15) and r + 1 (lanes 16-31) — so every HMMA A operand
      // is one load's four consecutive registers
      auto load_q = [&](int r, uint32_t* f) {
        ldsm_x4(plane + (uint32_t)((r * P + (int)lsel - 1 + (int)lrow) * 16), f[0], f[1], f[2], f[3]);
      };
      auto load_p = [&](int r, uint32_t* f) {
        ldsm_x4(plane + (uint32_t)((r * P + P * (int)lsel + 1 + (int)lrow) * 16), f[0], f[1], f[2], f[3]);
      };
      __half2 pool = zero2;
      // h2 rows go straight to the L2-resident workspace in the projection's
      // A layout [tile][group][row][16 B]: per warp store, 8 rows x 4 lanes x
      // 4 B = two whole 128-byte lines
      // (P = 8: into the resident compact h2: [chunk][group][64 rows][16 B])
      // (S2: the blurred 7x7 h2 to the workspace in the same compact layout)
      uint8_t* h2c = P == 8 ? smem + a.s_h2 + j * 8192 + g * 1024 + tq * 4
                     : S2   ? a.h2 + ((size_t)img * nch + j) * 8192 + g * 1024 + tq * 4
                            : h2img + (size_t)j * NT * 16384 + g * 2048 + tq * 4;
      // S2: output row yo of the Triangle-3 blur from conv rows 2 yo - 1 (kept
      // from the previous pair; row 1 reflected for yo = 0), 2 yo and 2 yo + 1;
      // along W the lane holding column 2 xo (flat i = 2 xo + 1) combines its
      // shuffled neighbours (column -1 reflects to 1)
      float2 po0 = make_float2(0.f, 0.f), po1 = make_float2(0.f, 0.f);
      auto epi_s2 = [&](int yo, const float* c0, const float* c1, const float* d0, const float* d1) {
        const float2 e0 = __half22float2(__hmul2(act_h2<ACT>(__floats2half2_rn(c0[0] + c1[0], c0[1] + c1[1])), m0));
        const float2 e1 = __half22float2(__hmul2(act_h2<ACT>(__floats2half2_rn(c0[2] + c1[2], c0[3] + c1[3])), m1));
        const float2 o0 = __half22float2(__hmul2(act_h2<ACT>(__floats2half2_rn(d0[0] + d1[0], d0[1] + d1[1])), m0));
        const float2 o1 = __half22float2(__hmul2(act_h2<ACT>(__floats2half2_rn(d0[2] + d1[2], d0[3] + d1[3])), m1));
        const float2 p0 = yo == 0 ? o0 : po0, p1 = yo == 0 ? o1 : po1;
        const float2 v0 = make_float2(0.25f * p0.x + 0.5f * e0.x + 0.25f * o0.x, 0.25f * p0.y + 0.5f * e0.y + 0.25f * o0.y);
        const float2 v1 = make_float2(0.25f * p1.x + 0.5f * e1.x + 0.25f * o1.x, 0.25f * p1.y + 0.5f * e1.y + 0.25f * o1.y);
        po0 = o0;
        po1 = o1;
        auto shf = [](float2 v, int src) {
          return make_float2(__shfl_sync(0xffffffffu, v.x, src), __shfl_sync(0xffffffffu, v.y, src));
        };
        const float2 up0 = shf(v0, (lane - 4) & 31), dn0 = shf(v0, (lane + 4) & 31);
        const float2 up1 = shf(v1, (lane - 4) & 31), dn1 = shf(v1, (lane + 4) & 31);
        const float2 first1 = shf(v1, tq);  // flat i = 8 (column 7)
        // columns 0..7 (i = gid, gid odd -> xo = (gid - 1) / 2)
        const float2 l0 = gid == 1 ? dn0 : up0, r0 = gid == 7 ? first1 : dn0;
        // columns 8..13 (i = gid + 8, gid in {1, 3, 5} -> xo = 4, 5, 6)
        const __half2 z0 = __floats2half2_rn(0.25f * l0.x + 0.5f * v0.x + 0.25f * r0.x,
                                             0.25f * l0.y + 0.5f * v0.y + 0.25f * r0.y);
        const __half2 z1 = __floats2half2_rn(0.25f * up1.x + 0.5f * v1.x + 0.25f * dn1.x,
                                             0.25f * up1.y + 0.5f * v1.y + 0.25f * dn1.y);
        if (gid & 1) {
          *reinterpret_cast<__half2*>(h2c + (8 * yo + (gid - 1) / 2 + 1) * 16) = z0;
          pool = __hadd2(pool, z0);
          if (gid < 7) {
            *reinterpret_cast<__half2*>(h2c + (8 * yo + (gid + 7) / 2 + 1) * 16) = z1;
            pool = __hadd2(pool, z1);
          }
        }
      };
      // fragment f = flat rows 16 f .. 16 f + 15; v1: its rows gid + 8 are image pixels
      auto epi = [&](int f, const float* c0, const float* c1, bool v1) {
        const __half2 h0 = __hmul2(act_h2<ACT>(__floats2half2_rn(c0[0] + c1[0], c0[1] + c1[1])), m0);
        const __half2 h1v = __hmul2(act_h2<ACT>(__floats2half2_rn(c0[2] + c1[2], c0[3] + c1[3])), v1 ? m1 : zero2);
        pool = __hadd2(pool, __hadd2(h0, h1v));
        if constexpr (P == 8) {
          const int fr = f * 16 + gid;  // flat row = compact A row
          *reinterpret_cast<__half2*>(h2c + fr * 16) = h0;
          *reinterpret_cast<__half2*>(h2c + (fr + 8) * 16) = h1v;
        } else {
          const int mm = f * 16 + gid;
          *reinterpret_cast<__half2*>(h2c + (mm >> 7) * 16384 + ((mm & 127) >> 3) * 128 + (mm & 7) * 16) = h0;
          const int m8 = mm + 8;
          *reinterpret_cast<__half2*>(h2c + (m8 >> 7) * 16384 + ((m8 & 127) >> 3) * 128 + (m8 & 7) * 16) = h1v;
        }
      };
      if constexpr (P == 16) {
      uint32_t Q0[4], Q1[4], Q2[4], Q3[4], P0[4], P1[4], P2[4], P3[4];
      // output row y: Q_y.(t0,t1) + Q_{y+1}.(t3,t4) + Q_{y+2}.(t6,t7) + P_y.(t2,t5) + P_{y+2}[0:2].t8
      load_q(0, Q0);
      load_q(1, Q1);
      load_p(0, P0);
      load_p(1, P1);
#pragma unroll
      for (int y = 0; y + 1 < H; y += 2) {
        load_q(y + 2, Q2);
        load_p(y + 2, P2);
        load_q(y + 3, Q3);
        load_p(y + 3, P3);
        float a0[4] = {bc.x, bc.y, bc.x, bc.y}, a1[4] = {0.f, 0.f, 0.f, 0.f};
        float b0[4] = {bc.x, bc.y, bc.x, bc.y}, b1[4] = {0.f, 0.f, 0.f, 0.f};
        hmma16(a0, Q0[0], Q0[1], Q0[2], Q0[3], bw[0], bw[1]);
        hmma16(b0, Q1[0], Q1[1], Q1[2], Q1[3], bw[0], bw[1]);
        hmma16(a1, P0[0], P0[1], P0[2], P0[3], bw[6], bw[7]);
        hmma16(b1, P1[0], P1[1], P1[2], P1[3], bw[6], bw[7]);
        hmma16(a0, Q1[0], Q1[1], Q1[2], Q1[3], bw[2], bw[3]);
        hmma16(b0, Q2[0], Q2[1], Q2[2], Q2[3], bw[2], bw[3]);
        hmma16(a1, Q2[0], Q2[1], Q2[2], Q2[3], bw[4], bw[5]);
        hmma16(b1, Q3[0], Q3[1], Q3[2], Q3[3], bw[4], bw[5]);
        hmma8(a0, P2[0], P2[1], bw[8]);
        hmma8(b0, P3[0], P3[1], bw[8]);
        if constexpr (S2) {
          epi_s2(y >> 1, a0, a1, b0, b1);
        } else {
          epi(y, a0, a1, true);
          epi(y + 1, b0, b1, true);
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          Q0[k] = Q2[k];
          Q1[k] = Q3[k];
          P0[k] = P2[k];
          P1[k] = P3[k];
        }
      }
      if constexpr (H % 2) {
        constexpr int y = H - 1;
        load_q(y + 2, Q2);
        load_p(y + 2, P2);
        float a0[4] = {bc.x, bc.y, bc.x, bc.y}, a1[4] = {0.f, 0.f, 0.f, 0.f}, a2[4] = {0.f, 0.f, 0.f, 0.f};
        hmma16(a0, Q0[0], Q0[1], Q0[2], Q0[3], bw[0], bw[1]);
        hmma16(a1, P0[0], P0[1], P0[2], P0[3], bw[6], bw[7]);
        hmma16(a2, Q1[0], Q1[1], Q1[2], Q1[3], bw[2], bw[3]);
        hmma16(a0, Q2[0], Q2[1], Q2[2], Q2[3], bw[4], bw[5]);
        hmma8(a1, P2[0], P2[1], bw[8]);
#pragma unroll
        for (int k = 0; k < 4; ++k) a1[k] += a2[k];
        epi(y, a0, a1, true);
      }
      } else {
      // P = 8: fragment f covers image rows 2f, 2f + 1 and reads units
      // s = 2f (dy = -1), 2f + 1 (dy = 0), 2f + 2 (dy = +1):
      //   Q_s.(t0,t1) + Q_{s+1}.(t3,t4) + Q_{s+2}.(t6,t7) + P_s.(t2,t5) + P_{s+2}[0:2].t8
      constexpr int NF = (P * H + 15) / 16;
      uint32_t Q0[4], Q1[4], Q2[4], Q3[4], Q4[4], P0[4], P1[4], P2[4];
      load_q(0, Q0);
      load_p(0, P0);
#pragma unroll
      for (int f = 0; f + 1 < NF; f += 2) {
        const int s0 = 2 * f;
        load_q(s0 + 1, Q1);
        load_q(s0 + 2, Q2);
        load_p(s0 + 2, P1);
        load_q(s0 + 3, Q3);
        load_q(s0 + 4, Q4);
        load_p(s0 + 4, P2);
        float a0[4] = {bc.x, bc.y, bc.x, bc.y}, a1[4] = {0.f, 0.f, 0.f, 0.f};
        float b0[4] = {bc.x, bc.y, bc.x, bc.y}, b1[4] = {0.f, 0.f, 0.f, 0.f};
        hmma16(a0, Q0[0], Q0[1], Q0[2], Q0[3], bw[0], bw[1]);
        hmma16(b0, Q2[0], Q2[1], Q2[2], Q2[3], bw[0], bw[1]);
        hmma16(a1, P0[0], P0[1], P0[2], P0[3], bw[6], bw[7]);
        hmma16(b1, P1[0], P1[1], P1[2], P1[3], bw[6], bw[7]);
        hmma16(a0, Q1[0], Q1[1], Q1[2], Q1[3], bw[2], bw[3]);
        hmma16(b0, Q3[0], Q3[1], Q3[2], Q3[3], bw[2], bw[3]);
        hmma16(a1, Q2[0], Q2[1], Q2[2], Q2[3], bw[4], bw[5]);
        hmma16(b1, Q4[0], Q4[1], Q4[2], Q4[3], bw[4], bw[5]);
        hmma8(a0, P1[0], P1[1], bw[8]);
        hmma8(b0, P2[0], P2[1], bw[8]);
        epi(f, a0, a1, 2 * f + 1 < H);
        epi(f + 1, b0, b1, 2 * f + 3 < H);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          Q0[k] = Q4[k];
          P0[k] = P2[k];
        }
      }
      if constexpr (NF % 2) {
        constexpr int f = NF - 1, s0 = 2 * f;
        load_q(s0 + 1, Q1);
        load_q(s0 + 2, Q2);
        load_p(s0 + 2, P1);
        float a0[4] = {bc.x, bc.y, bc.x, bc.y}, a1[4] = {0.f, 0.f, 0.f, 0.f}, a2[4] = {0.f, 0.f, 0.f, 0.f};
        hmma16(a0, Q0[0], Q0[1], Q0[2], Q0[3], bw[0], bw[1]);
        hmma16(a1, P0[0], P0[1], P0[2], P0[3], bw[6], bw[7]);
        hmma16(a2, Q1[0], Q1[1], Q1[2], Q1[3], bw[2], bw[3]);
        hmma16(a0, Q2[0], Q2[1], Q2[2], Q2[3], bw[4], bw[5]);
        hmma8(a1, P1[0], P1[1], bw[8]);
#pragma unroll
        for (int k = 0; k < 4; ++k) a1[k] += a2[k];
        epi(f, a0, a1, 2 * f + 1 < H);
      }
      }
      if (tid == 0) MB1_TRACE(28 + j);
      mbar_arrive(&B.h1_empty[b]);  // every ldmatrix of this buffer has completed (results consumed)
      if (j + 1 < nch) {
#pragma unroll
        for (int tp = 0; tp < 9; ++tp) bw[tp] = bwn[tp];
      }
      if (tid == 0) MB1_TRACE(20 + j);
      // SE pool of the chunk (fp16 per lane over <= 2H rows, fp32 across lanes):
      // reduce the 8 rows (gid) sharing a channel pair; the sums go to shared
      // memory for the E warps' squeeze
      const float2 pf = __half22float2(pool);
      float p0 = pf.x, p1 = pf.y;
#pragma unroll
      for (int sh = 4; sh < 32; sh <<= 1) {
        p0 += __shfl_xor_sync(0xffffffffu, p0, sh);
        p1 += __shfl_xor_sync(0xffffffffu, p1, sh);
      }
      if (gid == 0)
        *reinterpret_cast<float2*>(reinterpret_cast<float*>(s_se) + j * kHC + g * 8 + tq * 2) = make_float2(p0, p1);
      mbar_arrive(&B.pool_full[b]);
      if (tid == 0) MB1_TRACE(44 + j);
    }
    // the producer reloads h2 through the async proxy: order every thread's
    // generic-proxy stores before it
    if constexpr (P == 16) asm volatile("fence.proxy.async.global;" ::: "memory");
    float* scr = reinterpret_cast<float*>(s_se + hid * 4 + hid * 2);
    nbar(1, 256);
    if (tid == 0) mbar_arrive(&B.a_done);  // pool sums complete: the E warps squeeze
    MB1_TRACE(1);
    // ------------------------------------------------ phase B: excite
    __half2* s_gate = reinterpret_cast<__half2*>(s_se + hid * 4);
    const __half2* wex = reinterpret_cast<const __half2*>(s_wex);  // prefetched by the producer
    const float* bex = reinterpret_cast<const float*>(wp + a.o_se + a.o_bex);
    mbar_wait(&B.se_full, blk & 1);
    mbar_wait(&B.sq_full, blk & 1);
    {
      const float* s_s = scr + 256;
      for (int hp = tid; hp < hid / 2; hp += 256) {
        float e0, e1;
        if (hp == tid) {
          e0 = bex_pre.x;
          e1 = bex_pre.y;
        } else {
          e0 = bex[2 * hp];
          e1 = bex[2 * hp + 1];
        }
#pragma unroll 8
        for (int jj = 0; jj < sq; ++jj) {
          const float2 w = __half22float2(wex[(size_t)jj * (hid / 2) + hp]);
          e0 += s_s[jj] * w.x;
          e1 += s_s[jj] * w.y;
        }
        s_gate[hp] = __floats2half2_rn(act<kSigmoid>(e0), act<kSigmoid>(e1));
      }
      nbar(1, 256);
    }
    MB1_TRACE(2);
    // ------------------------------------------------ phase C: gate h2 chunks
    if constexpr (P == 8) {
      // the resident h2 ([chunk][group][64 rows][16 B]) gated in place chunk by
      // chunk, each released to the projection MMAs as soon as it is done
      uint4* h2s = reinterpret_cast<uint4*>(smem + a.s_h2);
      for (int jj = 0; jj < nch; ++jj) {
        const int gq = blk * nch + jj;
        // an arrival may not run a full phase ahead of the MMA's wait: chunk
        // jj - 4 (same barrier) must have been consumed
        mbar_wait(&B.pa_empty[gq & 3], ((gq >> 2) & 1) ^ 1);
#pragma unroll
        for (int k = 0; k < 2; ++k) {
          const int id = jj * 512 + k * 256 + tid, gg = (id >> 6) & 7;
          uint4 hv = h2s[id];
          const uint4 gv = *reinterpret_cast<const uint4*>(s_gate + jj * (kHC / 2) + gg * 4);
          __half2* h = reinterpret_cast<__half2*>(&hv);
          const __half2* gt = reinterpret_cast<const __half2*>(&gv);
#pragma unroll
          for (int i = 0; i < 4; ++i) h[i] = __hmul2(h[i], gt[i]);
          h2s[id] = hv;
        }
        fence_async_smem();
        mbar_arrive(&B.pa_ready[gq & 3]);
      }
    } else if constexpr (S2) {
      // each reloaded 7x7 chunk ([group][64 rows][16 B]) gated in its ring slot
      for (int jj = 0; jj < nch; ++jj) {
        const int gq = blk * nch + jj, s = gq & 3;
        mbar_wait(&B.pa_full[s], (gq >> 2) & 1);
        uint4* hs = reinterpret_cast<uint4*>(s_h1 + s * a.slot_bytes);
#pragma unroll
        for (int k = 0; k < 2; ++k) {
          const int id = k * 256 + tid, gg = id >> 6;
          uint4 hv = hs[id];
          const uint4 gv = *reinterpret_cast<const uint4*>(s_gate + jj * (kHC / 2) + gg * 4);
          __half2* h = reinterpret_cast<__half2*>(&hv);
          const __half2* gt = reinterpret_cast<const __half2*>(&gv);
#pragma unroll
          for (int i = 0; i < 4; ++i) h[i] = __hmul2(h[i], gt[i]);
          hs[id] = hv;
        }
        fence_async_smem();
        mbar_arrive(&B.pa_ready[s]);
      }
    } else {
    for (int qq = 0; qq < 2 * nch; ++qq) {
      const int gq = blk * 2 * nch + qq;
      const int s = gq & 3, u = gq >> 2, j = qq >> 1, half = qq & 1;
      mbar_wait(&B.pa_full[s], u & 1);
      // the gate scales W_prj's rows instead of h2: Z = h2 (diag(g) W_prj) touches the
      // slot's W half (4 K-core columns of C 16-byte units: 8 KB at C = 128) instead of
      // NT x 8 KB of h2 — half the shared-memory traffic of the gating pass
      uint8_t* slot = s_h1 + s * a.slot_bytes + NT * 8192;
#pragma unroll
      for (int k = 0; k < 4 * C / 256; ++k) {
        const int id = tid + k * 256;  // 16-byte unit: K-core column gg (8 hidden channels), output row
        const int gg = id / C;
        uint8_t* p = slot + id * 16;
        uint4 hv = lds128(p);
        const uint4 gv = *reinterpret_cast<const uint4*>(s_gate + j * (kHC / 2) + (half * 4 + gg) * 4);
        __half2* h = reinterpret_cast<__half2*>(&hv);
        const __half2* gt = reinterpret_cast<const __half2*>(&gv);
#pragma unroll
        for (int i = 0; i < 4; ++i) h[i] = __hmul2(h[i], gt[i]);
        *reinterpret_cast<uint4*>(p) = hv;
      }
      fence_async_smem();
      mbar_arrive(&B.pa_ready[s]);
    }
    }
    MB1_TRACE(3);
    }  // blocks
  }
  tc_fence_before();
  __syncthreads();
  if (warp == kMma) {
    __syncwarp();
    tmem_dealloc_n(tmem, a.tmem_cols);
  }
}


// =================================================================== host
}  // namespace wl

#include <algorithm>
#include <cstdlib>
#include "launch.h"

namespace wl {
long long* g_mb1_trace = nullptr;
void mb1_set_trace(void* p) { g_mb1_trace = reinterpret_cast<long long*>(p); }

namespace {
constexpr int kSmemMax1 = 232448;
constexpr int kWsHeader1 = 4096;  // the arrival-counter header every family leaves alone

bool mb1_plan(const wl_block_desc& d, Mb1Args& a) {
  memset(&a, 0, sizeof(a));
  a.n = d.n;
  a.H = d.h;
  a.W = d.w;
  a.C = d.c;
  a.K = d.stride == 2 ? d.k : d.c;
  const bool s2 = d.stride == 2;
  a.hid = d.expansion * d.c;
  a.sq = d.se_sq;
  a.nch = a.hid / mb1::kHC;
  a.NT = (mb1_pitch(a.H) * a.H + 127) / 128;
  const int C = a.C, hid = a.hid, NT = a.NT;
  const int GS = mb1_plane_bytes(a.H);
  // shared memory: x (swizzled halves) | h1 x2 | W_exp ring x2 (the phase C ring overlays h1 + ring) | hdr | SE | bars
  int o = 0;
  a.s_x = o;
  o += (C / 64) * NT * 128 * 128;
  a.s_h1_bytes = 2 * 8 * GS;
  const bool p8 = mb1_pitch(a.H) == 8;
  // phase C ring slot: P = 16: h2 half-chunk (NT x 8 KB) + W_prj half-chunk;
  // P = 8 (h2 resident): one W_prj chunk (C x 64 x 2)
  // S2: one 7x7 h2 chunk (8 KB) + one W_prj chunk (K x 64 x 2)
  a.slot_bytes = p8 ? C * mb1::kHC * 2 : s2 ? 8192 + a.K * mb1::kHC * 2 : NT * 8192 + C * 32 * 2;
  const int wring = 2 * mb1::kHC * C * 2;
  if (p8) {
    // W_exp ring | h1 (>= 2 slots): the phase C ring's slots 0 / 1 are the W_exp
    // buffers (free once the last two expands complete, before the conv ends),
    // slots 2 / 3 the h1 buffers (free after phase A); the block's h2 stays resident
    if (wring != 2 * a.slot_bytes || a.nch % 4) return false;
    a.s_w = o;
    o += wring;
    a.s_h1 = o;
    o = align_up(o + std::max(a.s_h1_bytes, 2 * a.slot_bytes), 1024);
    a.s_h2 = o;
    o += a.nch * 8192;
  } else {
    // the phase C ring (4 slots) overlays h1 + the W_exp ring: pad h1 when it is smaller
    a.s_h1 = o;
    o = align_up(o + std::max(a.s_h1_bytes, 4 * a.slot_bytes - wring), 128);
    a.s_w = o;
    o += wring;
    if (4 * a.slot_bytes > o - a.s_h1) return false;
  }
  a.o_bexp = 0;
  a.o_bconv = hid * 4;
  a.o_bprj = 2 * hid * 4;
  a.hdr_bytes = align_up(2 * hid * 4 + a.K * 4, 16);
  a.s_hdr = align_up(o, 128);
  a.hdr_stride = align_up(a.hdr_bytes, 128);
  o = a.s_hdr + 2 * a.hdr_stride;
  a.s_se = align_up(o, 128);
  o = a.s_se + hid * 4 + hid * 2 + (256 + 32) * 4;
  a.s_wex = align_up(o, 128);
  o = a.s_wex + a.sq * hid * 2;
  a.s_bar = align_up(o, 128);
  a.smem = a.s_bar + align_up((int)sizeof(mb1::Bars), 16);
  // packed blob
  int64_t p = a.hdr_bytes;
  a.o_se = p;
  int se = hid * 32 * 2;  // W_sq transposed: [32 squeeze outputs (zero past sq)][hid]
  a.o_bsq = align_up(se, 16);
  se = a.o_bsq + a.sq * 4;
  a.o_wex = align_up(se, 16);
  se = a.o_wex + a.sq * hid * 2;
  a.o_bex = align_up(se, 16);
  se = a.o_bex + hid * 4;
  p += align_up(se, 128);
  a.o_frag = p;
  p += (int64_t)a.nch * 8 * 9 * 32 * 4;
  a.o_wexp = p;
  p += (int64_t)a.nch * mb1::kHC * C * 2;
  a.o_wprj = p;
  a.t_e = 0;
  a.t_z = 2 * NT * mb1::kHC;
  const int cols = a.t_z + (s2 ? a.K : NT * C);
  a.tmem_cols = 32;
  while (a.tmem_cols < cols) a.tmem_cols *= 2;
  return a.smem <= kSmemMax1 && cols <= 512;
}
int64_t mb1_blob_bytes(const Mb1Args& a) { return a.o_wprj + (int64_t)a.nch * a.K * mb1::kHC * 2; }

static bool env_legacy() {
  static const bool v = getenv("WL_MB_LEGACY") != nullptr;  // A/B: force the block-diagonal tcgen05 conv kernel
  return v;
}

using Mb1K = void (*)(const CUtensorMap, const CUtensorMap, const Mb1Args);
template <int C, int ACT>
Mb1K mb1_pick_h(int h, bool s2) {
  if (s2) return h == 14 ? mb_s1_kernel<14, C, ACT, true> : nullptr;
  switch (h) {
    case 7: return mb_s1_kernel<7, C, ACT, false>;
    case 8: return mb_s1_kernel<8, C, ACT, false>;
    case 14: return mb_s1_kernel<14, C, ACT, false>;
    case 16: return mb_s1_kernel<16, C, ACT, false>;
  }
  return nullptr;
}
Mb1K mb1_kernel(const wl_block_desc& d) {
  const bool s2 = d.stride == 2;
  if (d.c == 128) return d.act == kSilu ? mb1_pick_h<128, kSilu>(d.h, s2) : mb1_pick_h<128, kRelu>(d.h, s2);
  if (d.c == 64) return d.act == kSilu ? mb1_pick_h<64, kSilu>(d.h, s2) : mb1_pick_h<64, kRelu>(d.h, s2);
  return nullptr;
}
}  // namespace

bool mb1_eligible(const wl_block_desc& d) {
  if (env_legacy() || d.kind != WL_KIND_MBCONV || d.group_width != 8) return false;
  if (d.stride == 1 && d.k != d.c) return false;
  // stride 2: the 14x14 -> 7x7 block (conv at 14x14, blur-pool, 7x7 tail)
  if (d.stride == 2 && (d.h != 14 || d.w != 14 || (d.k != 64 && d.k != 128))) return false;
  if (d.stride != 1 && d.stride != 2) return false;
  if ((d.c != 64 && d.c != 128) || d.w > 14 || d.w > mb1_pitch(d.h) - 1 || (d.act != kSilu && d.act != kRelu))
    return false;
  const int hid = d.expansion * d.c;
  if (hid % mb1::kHC || d.se_sq < 1 || d.se_sq > 32 || hid / 2 > 256 * 4) return false;
  Mb1Args a;
  return mb1_plan(d, a) && mb1_kernel(d) != nullptr;
}

int64_t mb1_packed_bytes(const wl_block_desc& d) {
  Mb1Args a;
  mb1_plan(d, a);
  return mb1_blob_bytes(a);
}

int64_t mb1_workspace(const wl_block_desc& d) {
  Mb1Args a;
  mb1_plan(d, a);
  return kWsHeader1 + (int64_t)d.n * a.nch * (d.stride == 2 ? 8192 : a.NT * 16384);
}

int mb1_pack(const wl_block_desc& d, const float* const* w, uint8_t* out) {
  Mb1Args a;
  mb1_plan(d, a);
  memset(out, 0, (size_t)mb1_blob_bytes(a));
  const int C = a.C, hid = a.hid, sq = a.sq, HC = mb1::kHC;
  const float *wexp = w[0], *bexp = w[1], *wconv = w[2], *bconv = w[3], *wsq = w[4], *bsq = w[5], *wex = w[6],
              *bex = w[7], *wprj = w[8], *bprj = w[9];
  float* hb = reinterpret_cast<float*>(out);
  for (int i = 0; i < hid; ++i) {
    hb[i] = bexp[i];
    hb[hid + i] = bconv[i];
  }
  const int K = a.K;
  for (int i = 0; i < K; ++i) hb[2 * hid + i] = bprj[i];
  uint8_t* se = out + a.o_se;
  for (int o = 0; o < sq; ++o)  // transposed [o][hid]; rows sq..31 stay zero
    for (int i = 0; i < hid; ++i) put_h(se, ((size_t)o * hid + i) * 2, wsq[(size_t)i * sq + o]);
  for (int i = 0; i < sq; ++i) reinterpret_cast<float*>(se + a.o_bsq)[i] = bsq[i];
  for (int i = 0; i < sq * hid; ++i) put_h(se + a.o_wex, (size_t)i * 2, wex[i]);
  for (int i = 0; i < hid; ++i) reinterpret_cast<float*>(se + a.o_bex)[i] = bex[i];
  // mma.sync B fragments: [chunk][group][slot][lane] = (w[co][tap][ci], w[co][tap][ci + 1]),
  // co = 8 G + lane / 4, ci = 2 (lane % 4)   (w_conv is (hid, 3, 3, T=8)); slots
  // hold the taps in k16-pair order (0,1) (3,4) (6,7) (2,5) 8
  static const int kTapOfSlot[9] = {0, 1, 3, 4, 6, 7, 2, 5, 8};
  uint8_t* fr = out + a.o_frag;
  for (int G = 0; G < hid / 8; ++G)
    for (int slot = 0; slot < 9; ++slot)
      for (int l = 0; l < 32; ++l) {
        const int tap = kTapOfSlot[slot];
        const int co = 8 * G + l / 4, ci = 2 * (l % 4);
        const size_t off = (((size_t)G * 9 + slot) * 32 + l) * 4;
        put_h(fr, off, wconv[((size_t)co * 9 + tap) * 8 + ci]);
        put_h(fr, off + 2, wconv[((size_t)co * 9 + tap) * 8 + ci + 1]);
      }
  // W_exp chunk j: B operand (N = 64 hidden x K = C), 8x8 core matrices, LBO 1024
  for (int j = 0; j < a.nch; ++j) {
    uint8_t* ch = out + a.o_wexp + (size_t)j * HC * C * 2;
    for (int nn = 0; nn < HC; ++nn)
      for (int k = 0; k < C; ++k) put_h(ch, core_off_h(nn, k, 1024), wexp[(size_t)k * hid + j * HC + nn]);
  }
  // W_prj chunk j: B operand (N = K output channels x K = 64 hidden), LBO = (K / 8) 128
  for (int j = 0; j < a.nch; ++j) {
    uint8_t* ch = out + a.o_wprj + (size_t)j * K * HC * 2;
    for (int nn = 0; nn < K; ++nn)
      for (int k = 0; k < HC; ++k) put_h(ch, core_off_h(nn, k, (K / 8) * 128), wprj[(size_t)(j * HC + k) * K + nn]);
  }
  return WL_OK;
}

static int mb1_launch(const wl_block_desc& d, Mb1Args& a, const void* x, void* z, cudaStream_t st) {
  CUtensorMap tx, tz;
  const uint64_t dims[4] = {(uint64_t)d.c, (uint64_t)d.w, (uint64_t)d.h, (uint64_t)d.n};
  const uint64_t strides[3] = {(uint64_t)d.c * 2, (uint64_t)d.w * d.c * 2, (uint64_t)d.h * d.w * d.c * 2};
  // P = 8: one box per pair of image rows (a 16-row fragment, placed at A rows 32 k)
  const uint32_t box[4] = {64, (uint32_t)mb1_pitch(d.h), mb1_pitch(d.h) == 8 ? 2u : (uint32_t)d.h, 1};
  if (int e = encode_tmap(&tx, x, 4, dims, strides, box, true)) return e;
  if (d.stride == 2) {
    // 7x7 output, stored as pairs of rows from the compact pitch-8 staging
    const uint64_t zd[4] = {(uint64_t)d.k, (uint64_t)(d.w / 2), (uint64_t)(d.h / 2), (uint64_t)d.n};
    const uint64_t zs[3] = {(uint64_t)d.k * 2, (uint64_t)(d.w / 2) * d.k * 2, (uint64_t)(d.h / 2) * (d.w / 2) * d.k * 2};
    const uint32_t zb[4] = {64, 8, 2, 1};
    if (int e = encode_tmap(&tz, z, 4, zd, zs, zb, true)) return e;
  } else if (int e = encode_tmap(&tz, z, 4, dims, strides, box, true)) {
    return e;
  }
  return launch_pdl(mb1_kernel(d), d.n, mb1::kThreads, a.smem, st, "mb_s1 launch", tx, tz, a);
}

int mb1_forward(const wl_block_desc& d, const void* x, const void* packed, void* z, void* ws, cudaStream_t st) {
  Mb1Args a;
  mb1_plan(d, a);
  a.wpack = reinterpret_cast<const uint8_t*>(packed);
  a.nblk = 1;
  a.h2 = reinterpret_cast<uint8_t*>(ws) + kWsHeader1;
  a.trace = g_mb1_trace;
  return mb1_launch(d, a, x, z, st);
}

int mb1_stage_max(const wl_block_desc& d) { return d.stride == 1 && mb1_eligible(d) ? kMb1MaxStage : 0; }

// nblk consecutive identical stride-1 MBConv blocks in one launch: the image
// stays in shared memory between blocks (the per-stage persistent kernel)
int mb1_stage_forward(const wl_block_desc& d, int nblk, const void* x, const void* const* packed, void* z, void* ws,
                      cudaStream_t st) {
  if (d.stride != 1 || !mb1_eligible(d))
    return set_error(WL_EUNSUPPORTED, "stage launch: block is not a stride-1 T=8 MBConv (W <= 14)");
  if (nblk < 1 || nblk > kMb1MaxStage)
    return set_error(WL_EUNSUPPORTED, "stage launch: 1..%d blocks (got %d)", kMb1MaxStage, nblk);
  Mb1Args a;
  mb1_plan(d, a);
  a.nblk = nblk;
  for (int i = 0; i < nblk; ++i) {
    if (!packed[i]) return set_error(WL_EINVAL, "stage launch: packed blob %d is null", i);
    a.wpacks[i] = reinterpret_cast<const uint8_t*>(packed[i]);
  }
  a.wpack = a.wpacks[0];
  a.h2 = reinterpret_cast<uint8_t*>(ws) + kWsHeader1;
  a.trace = g_mb1_trace;
  return mb1_launch(d, a, x, z, st);
}

int mb1_init() {
  for (int c : {64, 128})
    for (int act : {kSilu, kRelu})
      for (int h : {7, 8, 14, 16, -14}) {  // -14: the stride-2 14x14 -> 7x7 variant
        wl_block_desc d;
        memset(&d, 0, sizeof(d));
        d.c = c;
        d.act = act;
        d.h = h < 0 ? -h : h;
        d.stride = h < 0 ? 2 : 1;
        if (int e = check_cuda(cudaFuncSetAttribute(mb1_kernel(d), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                    kSmemMax1),
                               "cudaFuncSetAttribute(mb_s1)"))
          return e;
      }
  return WL_OK;
}

}  // namespace wl
