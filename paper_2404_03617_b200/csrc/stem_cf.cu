// stem_cf.cu — the network's first two units in one kernel: the dense 3x3
// stride-2 stem (+ ReLU, core.py:135-141; ops complexity.py:147-151) feeding
// the first stride-1 ConvFirst block (T = 8, C = 16; core.py:100-109, fused
// schedule machine.py:462-525). The stem output h never leaves the SM
// (PAPER.md:1763-1766): only the image and the block's
// output cross HBM.
//
// Everything is a small matrix, so the whole chain runs on the warp-level
// tensor path (mma.sync m16n8k16 / m16n8k8, fp32 accumulation) with the
// accumulators of one stage re-packed in registers as the A fragments of the
// next (the C-fragment -> A-fragment identity of m16n8k16):
//   per CTA tile of 8 x 16 output pixels:
//     TMA: the 21 x 37 x 3 input patch (zero outside the image), double-buffered
//     stem  : 180 h pixels (the tile + 1-pixel halo) = im2col(patch) . W_s (K 27 -> 32),
//             + b, ReLU -> two 8-channel h planes in shared memory (0 outside the image)
//     per warp = one output row of 16 pixels:
//       conv   : grouped 3x3, T = 8 (two groups), ldmatrix fragments of the flat
//                h planes (pitch 18: the +-1 taps are +-1 flat rows), 5 MMAs / group
//       expand : (conv + b_conv) . U (16 -> 48), + a, phi
//       project: . V (48 -> 16), + b + h (the residual), -> staged -> 512 B store
#include <cuda.h>
#include <cuda_fp16.h>
#include <cstdint>
#include <cstring>
#include "common.cuh"
#include "launch.h"
#include "plan.h"

namespace wl {

namespace scf {
constexpr int kThreads = 256;  // 8 warps = 8 output rows of 16 pixels
constexpr int kTY = 8, kTX = 16;
constexpr int kPR = 2 * kTY + 5, kPC = 120;  // patch rows, patch row pitch (halves): 7 + 37 x 3 -> 120
constexpr int kPatch = (kPR * kPC * 2 + 127) / 128 * 64;  // halves per patch buffer (128 B multiple)
constexpr int kHP = 18;                       // h plane pitch (pixels): the tile's 16 + 2 halo
constexpr int kHR = kTY + 2;                  // h plane rows
// packed blob (fp32 biases, then per-lane B fragments, uint32 each)
constexpr int kOffBs = 0, kOffBc = 16, kOffA = 32, kOffB = 80;  // floats
constexpr int kHdrFloats = 96;
constexpr int kFragStem = 2 * 2 * 2;   // n8 tiles x k16 steps x regs
constexpr int kFragConv = 2 * 9;       // groups x slots
constexpr int kFragU = 6 * 2;          // n8 tiles x regs
constexpr int kFragV = 2 * 3 * 2;      // n8 tiles x k16 steps x regs
constexpr int kFrags = kFragStem + kFragConv + kFragU + kFragV;  // 50 per lane
struct Args {
  int n, H, W;  // input image (H x W x 3); output (H/2) x (W/2) x 16
  int tiles_x, tiles_y, tiles;
  const uint8_t* wpack;
  __half* z;
};
}  // namespace scf

__device__ __forceinline__ void scf_hmma16(float* d, uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0,
                                           uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, "
      "{%0, %1, %2, %3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void scf_hmma8(float* d, uint32_t a0, uint32_t a1, uint32_t b0) {
  asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.f16.f16.f32 {%0, %1, %2, %3}, {%4, %5}, {%6}, {%0, %1, %2, %3};"
               : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
               : "r"(a0), "r"(a1), "r"(b0));
}
__device__ __forceinline__ void scf_ldsm4(uint32_t addr, uint32_t* r) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0, %1, %2, %3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr));
}
__device__ __forceinline__ uint32_t h2u(__half2 h) { return *reinterpret_cast<uint32_t*>(&h); }
__device__ __forceinline__ void scf_tma3(void* dst, const void* tmap, int c0, int c1, int c2, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
      "[%5];" ::"r"(smem_u32(dst)),
      "l"(tmap), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}

template <int ACT>
__global__ void __launch_bounds__(scf::kThreads, 2)
    stem_cf_kernel(const __grid_constant__ CUtensorMap tmap_x, const __grid_constant__ scf::Args a) {
  using namespace scf;
  __shared__ __align__(128) __half s_patch[2][kPatch];  // 128-byte aligned buffers
  __shared__ __align__(128) uint8_t s_h[2][kHR * kHP * 16];  // two 8-channel planes, 16 B per pixel
  __shared__ __align__(16) __half s_out[8][kTX * 16];
  __shared__ __align__(8) uint64_t bar[2];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gid = lane >> 2, tq = lane & 3;
  const int HO = a.H / 2, WO = a.W / 2;

  // ---- per-lane weights (B fragments) and biases
  const uint32_t* frag = reinterpret_cast<const uint32_t*>(a.wpack + kHdrFloats * 4) + lane * kFrags;
  uint32_t fs[kFragStem], fc[kFragConv], fu[kFragU], fv[kFragV];
#pragma unroll
  for (int i = 0; i < kFragStem; ++i) fs[i] = __ldg(frag + i);
#pragma unroll
  for (int i = 0; i < kFragConv; ++i) fc[i] = __ldg(frag + kFragStem + i);
#pragma unroll
  for (int i = 0; i < kFragU; ++i) fu[i] = __ldg(frag + kFragStem + kFragConv + i);
#pragma unroll
  for (int i = 0; i < kFragV; ++i) fv[i] = __ldg(frag + kFragStem + kFragConv + kFragU + i);
  const float* hdr = reinterpret_cast<const float*>(a.wpack);
  float bs[2][2], bc[2][2], ba[6][2], bb[2][2];
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    bs[j][0] = hdr[kOffBs + 8 * j + 2 * tq];
    bs[j][1] = hdr[kOffBs + 8 * j + 2 * tq + 1];
    bc[j][0] = hdr[kOffBc + 8 * j + 2 * tq];
    bc[j][1] = hdr[kOffBc + 8 * j + 2 * tq + 1];
    bb[j][0] = hdr[kOffB + 8 * j + 2 * tq];
    bb[j][1] = hdr[kOffB + 8 * j + 2 * tq + 1];
  }
#pragma unroll
  for (int j = 0; j < 6; ++j) {
    ba[j][0] = hdr[kOffA + 8 * j + 2 * tq];
    ba[j][1] = hdr[kOffA + 8 * j + 2 * tq + 1];
  }
  // im2col offsets of this lane's A-fragment columns: k = (kr * 3 + ks) * 3 + c
  int koff[2][4];  // [k16 step][k = 2tq, 2tq + 1, 2tq + 8, 2tq + 9]
#pragma unroll
  for (int s = 0; s < 2; ++s)
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int k = 16 * s + 2 * tq + (e & 1) + 8 * (e >> 1);
      const int kr = k / 9, ks = (k / 3) % 3, c = k % 3;
      // k >= 27 carries zero weights: any finite patch element will do
      koff[s][e] = k < 27 ? kr * kPC + ks * 3 + c : 0;
    }

  if (threadIdx.x == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_mbar_init();
  }
  __syncthreads();
  pdl_wait();
  const int my_tiles = blockIdx.x < a.tiles ? (a.tiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const int tpi = a.tiles_x * a.tiles_y;
  const float inv_tpi = 1.f / (float)tpi, inv_tx = 1.f / (float)a.tiles_x;
  // v / d for v < 2^24 by a float reciprocal and one correction step (every
  // warp derives its tile coordinates: two integer divisions were ~11% of the
  // kernel's instructions)
  auto fdiv = [](int v, int d, float inv) {
    int q = (int)((float)v * inv);
    if (q * d > v) --q;
    else if ((q + 1) * d <= v) ++q;
    return q;
  };
  auto tile_of = [&](int t, int& img, int& y0, int& x0) {
    const int tile = blockIdx.x + t * gridDim.x;
    img = fdiv(tile, tpi, inv_tpi);
    const int r = tile - img * tpi;
    const int ty = fdiv(r, a.tiles_x, inv_tx);
    y0 = ty * kTY;
    x0 = (r - ty * a.tiles_x) * kTX;
  };
  auto load_patch = [&](int t) {
    int img, y0, x0;
    tile_of(t, img, y0, x0);
    const int b = t & 1;
    mbar_arrive_expect_tx(&bar[b], kPR * kPC * 2);
    // the box must start on a 16-byte boundary of the innermost (w x c) dimension:
    // start 7 elements before pixel 2 x0 - 3 (x0 % 16 == 0 makes 6 x0 - 16 a multiple of 8)
    scf_tma3(s_patch[b], &tmap_x, 6 * x0 - 16, 2 * y0 - 3, img, &bar[b]);
  };
  if (threadIdx.x == 0 && my_tiles > 0) load_patch(0);

  for (int t = 0; t < my_tiles; ++t) {
    int img, y0, x0;
    tile_of(t, img, y0, x0);
    // the next tile's patch goes to the buffer tile t - 1 released (its stem
    // ended before the barrier that closed tile t - 1): a whole tile of lead
    if (threadIdx.x == 0 && t + 1 < my_tiles) load_patch(t + 1);
    const int pb = t & 1;
    mbar_wait(&bar[pb], (t >> 1) & 1);
    const __half* patch = s_patch[pb];
    // ------------------------------------------------------------ stem
    for (int mt = warp; mt < (kHR * kHP + 15) / 16; mt += 8) {
      const int p0 = mt * 16 + gid, p1 = p0 + 8;  // flat h pixels of this lane's two rows
      // rows past the plane gather from its last pixel (in bounds; results dropped)
      const int q0 = min(p0, kHR * kHP - 1), q1 = min(p1, kHR * kHP - 1);
      const int base0 = 2 * (q0 / kHP) * kPC + 2 * (q0 % kHP) * 3 + 7, base1 = 2 * (q1 / kHP) * kPC + 2 * (q1 % kHP) * 3 + 7;
      float acc[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
#pragma unroll
      for (int s = 0; s < 2; ++s) {
        __half e[2][4];  // [row][k]
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int o = koff[s][q];
          e[0][q] = patch[base0 + o];
          e[1][q] = patch[base1 + o];
        }
        const uint32_t a0 = h2u(__halves2half2(e[0][0], e[0][1])), a1 = h2u(__halves2half2(e[1][0], e[1][1]));
        const uint32_t a2 = h2u(__halves2half2(e[0][2], e[0][3])), a3 = h2u(__halves2half2(e[1][2], e[1][3]));
#pragma unroll
        for (int j = 0; j < 2; ++j) scf_hmma16(acc[j], a0, a1, a2, a3, fs[(j * 2 + s) * 2], fs[(j * 2 + s) * 2 + 1]);
      }
      // + b, ReLU; zero outside the image (the block's conv pads h with zeros)
#pragma unroll
      for (int rr = 0; rr < 2; ++rr) {
        const int p = rr ? p1 : p0;
        if (p >= kHR * kHP) continue;
        const int hy = y0 - 1 + p / kHP, hx = x0 - 1 + p % kHP;
        const bool in = hy >= 0 && hy < HO && hx >= 0 && hx < WO;
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const float f0 = fmaxf(acc[j][2 * rr] + bs[j][0], 0.f), f1 = fmaxf(acc[j][2 * rr + 1] + bs[j][1], 0.f);
          const __half2 h = in ? __floats2half2_rn(f0, f1) : __float2half2_rn(0.f);
          *reinterpret_cast<__half2*>(s_h[j] + p * 16 + tq * 4) = h;
        }
      }
    }
    __syncthreads();
    // ------------------------------------------- conv -> expand -> project
    {
      const int r = warp + 1;  // h plane row of this warp's output row
      const uint32_t lrow = lane & 15, lsel = lane >> 4;
      float cacc[2][4];
#pragma unroll
      for (int g = 0; g < 2; ++g) {
        const uint32_t plane = smem_u32(s_h[g]);
        // Q(rr): taps dx = -1 (lanes 0-15) and dx = 0 (lanes 16-31) of plane row rr;
        // P(rr): dx = +1 of rows rr (lanes 0-15) and rr + 1 (lanes 16-31)
        auto q_at = [&](int rr) { return plane + (uint32_t)((rr * kHP + 1 + (int)lrow - 1 + (int)lsel) * 16); };
        auto p_at = [&](int rr) { return plane + (uint32_t)(((rr + (int)lsel) * kHP + 1 + (int)lrow + 1) * 16); };
        uint32_t Q0[4], Q1[4], Q2[4], P0[4], P2[4];
        scf_ldsm4(q_at(r - 1), Q0);
        scf_ldsm4(q_at(r), Q1);
        scf_ldsm4(q_at(r + 1), Q2);
        scf_ldsm4(p_at(r - 1), P0);
        scf_ldsm4(p_at(r + 1), P2);
        float a0[4] = {0.f, 0.f, 0.f, 0.f}, a1[4] = {0.f, 0.f, 0.f, 0.f};
        const uint32_t* w = fc + 9 * g;
        scf_hmma16(a0, Q0[0], Q0[1], Q0[2], Q0[3], w[0], w[1]);  // (t0, t1)
        scf_hmma16(a1, P0[0], P0[1], P0[2], P0[3], w[6], w[7]);  // (t2, t5)
        scf_hmma16(a0, Q1[0], Q1[1], Q1[2], Q1[3], w[2], w[3]);  // (t3, t4)
        scf_hmma16(a1, Q2[0], Q2[1], Q2[2], Q2[3], w[4], w[5]);  // (t6, t7)
        scf_hmma8(a0, P2[0], P2[1], w[8]);                       // t8
#pragma unroll
        for (int i = 0; i < 4; ++i) cacc[g][i] = a0[i] + a1[i] + bc[g][i & 1];
      }
      // expand: A = conv output (16 px x 16 ch) from the two n8 accumulators
      const uint32_t xa0 = h2u(__floats2half2_rn(cacc[0][0], cacc[0][1]));
      const uint32_t xa1 = h2u(__floats2half2_rn(cacc[0][2], cacc[0][3]));
      const uint32_t xa2 = h2u(__floats2half2_rn(cacc[1][0], cacc[1][1]));
      const uint32_t xa3 = h2u(__floats2half2_rn(cacc[1][2], cacc[1][3]));
      uint32_t ha[6][2];  // phi(E + a) packed: [n8 tile][row gid | gid + 8]
#pragma unroll
      for (int j = 0; j < 6; ++j) {
        float e[4] = {0.f, 0.f, 0.f, 0.f};
        scf_hmma16(e, xa0, xa1, xa2, xa3, fu[2 * j], fu[2 * j + 1]);
        ha[j][0] = h2u(act_h2<ACT>(__floats2half2_rn(e[0] + ba[j][0], e[1] + ba[j][1])));
        ha[j][1] = h2u(act_h2<ACT>(__floats2half2_rn(e[2] + ba[j][0], e[3] + ba[j][1])));
      }
      // project: K = 48 in three k16 steps (n8 tiles 2s, 2s + 1 of the hidden)
      float z[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
#pragma unroll
      for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int s = 0; s < 3; ++s)
          scf_hmma16(z[j], ha[2 * s][0], ha[2 * s][1], ha[2 * s + 1][0], ha[2 * s + 1][1], fv[(j * 3 + s) * 2],
                     fv[(j * 3 + s) * 2 + 1]);
      // + b + residual h, stage the 16 x 16 row, one 512-byte store
#pragma unroll
      for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int rr = 0; rr < 2; ++rr) {
          const int px = gid + 8 * rr;
          const float2 res =
              __half22float2(*reinterpret_cast<const __half2*>(s_h[j] + (r * kHP + 1 + px) * 16 + tq * 4));
          const __half2 o = __floats2half2_rn(z[j][2 * rr] + bb[j][0] + res.x, z[j][2 * rr + 1] + bb[j][1] + res.y);
          *reinterpret_cast<__half2*>(&s_out[warp][px * 16 + 8 * j + 2 * tq]) = o;
        }
      __syncwarp();
      const int oy = y0 + warp;
      if (oy < HO) {
        const int px = lane >> 1, ox = x0 + px;
        if (ox < WO)
          *reinterpret_cast<uint4*>(a.z + (((size_t)img * HO + oy) * WO + ox) * 16 + (lane & 1) * 8) =
              *reinterpret_cast<const uint4*>(&s_out[warp][px * 16 + (lane & 1) * 8]);
      }
    }
    __syncthreads();  // h planes are rewritten by the next tile's stem
  }
  pdl_trigger();
}

// =================================================================== host
namespace {
using ScfK = void (*)(const CUtensorMap, const scf::Args);
ScfK scf_kernel(int act) { return act == kSilu ? stem_cf_kernel<kSilu> : stem_cf_kernel<kRelu>; }
}  // namespace

// stem (d0) followed by a stride-1 T=8 ConvFirst on its 16 output channels (d1)
bool stem_cf_supported(const wl_block_desc& d0, const wl_block_desc& d1) {
  return d0.kind == WL_KIND_STEM && d0.c == 3 && d0.k == 16 && d0.act == kRelu && d0.h % 2 == 0 && d0.w % 2 == 0 &&
         d0.h / 2 <= 4096 && d1.kind == WL_KIND_CONVFIRST && d1.stride == 1 && d1.group_width == 8 &&
         d1.ksize == 3 && d1.norm == WL_NORM_NONE && d1.c == 16 && d1.k == 16 && d1.expansion == 3 &&
         (d1.act == kRelu || d1.act == kSilu) && d1.n == d0.n && d1.h == d0.h / 2 && d1.w == d0.w / 2;
}
int64_t stem_cf_packed_bytes() { return (scf::kHdrFloats + 32 * scf::kFrags) * 4; }

// w0: stem (w_stem (16, 3, 3, 3), b_stem (16)); w1: ConvFirst (w_conv (16, 3, 3, 8),
// b_conv (16), u (16, 48), a (48), v (48, 16), b (16))
int stem_cf_pack(const float* const* w0, const float* const* w1, uint8_t* out) {
  using namespace scf;
  memset(out, 0, (size_t)stem_cf_packed_bytes());
  float* hdr = reinterpret_cast<float*>(out);
  for (int i = 0; i < 16; ++i) {
    hdr[kOffBs + i] = w0[1][i];
    hdr[kOffBc + i] = w1[1][i];
    hdr[kOffB + i] = w1[5][i];
  }
  for (int i = 0; i < 48; ++i) hdr[kOffA + i] = w1[3][i];
  uint8_t* fr = out + kHdrFloats * 4;
  auto put2 = [&](int lane, int idx, float lo, float hi) {
    put_h(fr, ((size_t)lane * kFrags + idx) * 4, lo);
    put_h(fr, ((size_t)lane * kFrags + idx) * 4 + 2, hi);
  };
  static const int kTapOfSlot[9] = {0, 1, 3, 4, 6, 7, 2, 5, 8};
  for (int l = 0; l < 32; ++l) {
    const int g = l >> 2, t2 = 2 * (l & 3);
    // stem B: K = im2col (27 -> 32), N = 16; reg (j, s, h) holds k = 16 s + t2 (+1) (+8 h)
    for (int j = 0; j < 2; ++j)
      for (int s = 0; s < 2; ++s)
        for (int h = 0; h < 2; ++h) {
          const int k = 16 * s + t2 + 8 * h, co = 8 * j + g;
          const float lo = k < 27 ? w0[0][co * 27 + k] : 0.f, hi = k + 1 < 27 ? w0[0][co * 27 + k + 1] : 0.f;
          put2(l, (j * 2 + s) * 2 + h, lo, hi);
        }
    // conv B (per group, mb_s1's slot order): (w[co][tap][ci], w[co][tap][ci + 1])
    for (int gg = 0; gg < 2; ++gg)
      for (int slot = 0; slot < 9; ++slot) {
        const int tap = kTapOfSlot[slot], co = 8 * gg + g;
        put2(l, kFragStem + 9 * gg + slot, w1[0][(co * 9 + tap) * 8 + t2], w1[0][(co * 9 + tap) * 8 + t2 + 1]);
      }
    // U (16 x 48): n8 tile j, k = t2 (+1) and t2 + 8 (+1)
    for (int j = 0; j < 6; ++j)
      for (int h = 0; h < 2; ++h) {
        const int k = t2 + 8 * h, n = 8 * j + g;
        put2(l, kFragStem + kFragConv + 2 * j + h, w1[2][k * 48 + n], w1[2][(k + 1) * 48 + n]);
      }
    // V (48 x 16): n8 tile j, k16 step s
    for (int j = 0; j < 2; ++j)
      for (int s = 0; s < 3; ++s)
        for (int h = 0; h < 2; ++h) {
          const int k = 16 * s + t2 + 8 * h, n = 8 * j + g;
          put2(l, kFragStem + kFragConv + kFragU + (j * 3 + s) * 2 + h, w1[4][k * 16 + n], w1[4][(k + 1) * 16 + n]);
        }
  }
  return WL_OK;
}

int stem_cf_forward(const wl_block_desc& d0, const wl_block_desc& d1, const void* x, const void* packed, void* z,
                    cudaStream_t st) {
  using namespace scf;
  if (!stem_cf_supported(d0, d1)) return set_error(WL_EUNSUPPORTED, "stem + ConvFirst pair: unsupported shapes");
  Args a;
  memset(&a, 0, sizeof(a));
  a.n = d0.n;
  a.H = d0.h;
  a.W = d0.w;
  a.tiles_x = (d0.w / 2 + kTX - 1) / kTX;
  a.tiles_y = (d0.h / 2 + kTY - 1) / kTY;
  a.tiles = a.n * a.tiles_x * a.tiles_y;
  a.wpack = reinterpret_cast<const uint8_t*>(packed);
  a.z = reinterpret_cast<__half*>(z);
  CUtensorMap tm;
  const uint64_t dims[3] = {(uint64_t)d0.w * 3, (uint64_t)d0.h, (uint64_t)d0.n};
  const uint64_t strides[2] = {(uint64_t)d0.w * 3 * 2, (uint64_t)d0.h * d0.w * 3 * 2};
  const uint32_t box[3] = {(uint32_t)kPC, (uint32_t)kPR, 1};
  if (int e = encode_tmap(&tm, x, 3, dims, strides, box)) return e;
  const int grid = a.tiles < 2 * kNumSMs ? a.tiles : 2 * kNumSMs;
  return launch_pdl(scf_kernel(d1.act), grid, kThreads, 0, st, "stem_cf launch", tm, a);
}

}  // namespace wl
